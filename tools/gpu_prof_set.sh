# ncu --set full of chosen kernels inside one warm (async) search:
#   c1: k_fuse_block, k_expand_filter (largest = generation 4), k_screen_static (gen 4)
#   c4 (2048 pairs): k_mscreen gen 5, k_mdecide gen 5
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
prof() {  # name cfg kernel skip extra...
  local name=$1 cfg=$2 k=$3 s=$4; shift 4
  timeout 900 ncu --nvtx --nvtx-include "prof/" --set full --clock-control none --import-source on \
    -k regex:^$k\$ -s $s -c 1 -f -o gpurun_out/prof_$name python tools/prof_search.py --config $cfg "$@" \
    > gpurun_out/ncu_$name.log 2>&1
  echo "$name rc=$?"; grep -E "error|ERROR" gpurun_out/ncu_$name.log | head -3
}
python tools/prof_search.py --config c1 > gpurun_out/plain_c1.log 2>&1 && echo plain ok
prof fuse c1 k_fuse_block 0
prof expand c1 k_expand_filter 4
prof static c1 k_screen_static 4
prof mscreen c4 k_mscreen 5 --pairs 2048
prof mdecide c4 k_mdecide 5 --pairs 2048
