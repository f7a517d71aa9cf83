# c1 bench (device value + screen breakdown) for the default library and every variants/lib_*.so
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CFG=${1:-c1}
for v in default variants/lib_*.so; do echo "== $v" >> gpurun_out/variants_summary.txt
  if [ "$v" = default ]; then unset LTSG_LIB; else export LTSG_LIB=$v; fi
  timeout 600 python bench.py --config $CFG --steps ${STEPS:-10} --warmup 3 --no-cpu --no-allpairs ${EXTRA:-} > gpurun_out/var.log 2>&1
  python - "$v" <<'PY'
import json,sys
d=json.loads(open('gpurun_out/var.log').read().strip().splitlines()[-1])
r=d.get('roofline',{})
open('gpurun_out/variants_summary.txt','a').write(' '.join([sys.argv[1], 'value %.3e'%d['value'], 'ms %.3f'%d['ms_per_step'], 'expand %.3f'%r.get('expand_ms_per_step',0), 'exact %.3f'%r.get('kernel_ms_per_step',0), 'screen %.3f'%r.get('screen_ms_per_step',0), 'fuse %.3f'%d['breakdown_ms_per_step']['contacts_fusion'], 'e2e %.3e'%d['e2e']['value']])+chr(10)); print(sys.argv[1], 'value %.3e'%d['value'], 'ms %.3f'%d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'], 'decided %d exact %d'%(r.get('bound_rows_per_step',0), r.get('exact_rows_per_step',0)), 'screen %.3f'%r.get('screen_ms_per_step',0), 'kernel %.3f'%r.get('kernel_ms_per_step',0), 'expand %.3f'%r.get('expand_ms_per_step',0), json.dumps(d.get('breakdown_ms_per_step')))
PY
done
