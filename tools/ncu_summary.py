"""Summarise an ncu report: key throughput metrics, stall reasons and the
per-opcode executed-instruction mix (from the SASS source page)."""
import csv
import re
import subprocess
import sys
from collections import Counter


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return [dict(zip(r[0], row)) for row in r[2:]], dict(zip(r[0], r[1]))


def source(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    hdr = r[1]
    return [dict(zip(hdr, row)) for row in r[2:] if len(row) == len(hdr) and row[0] != hdr[0]]


KEYS = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"]


def main(rep, rows=None):
    recs, units = raw(rep)
    for d in recs:
        print("kernel:", d.get("Kernel Name", "")[:80])
        for k in KEYS:
            print(f"  {k:70s} {d.get(k, '')} {units.get(k, '')}")
        st = []
        for k, v in d.items():
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
                try:
                    st.append((float(v), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        print("  stalls/issue:", ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:8]))
    src = source(rep)
    cnt, th = Counter(), Counter()
    for r in src:
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r.get("Source", ""))
        if not m:
            continue
        try:
            cnt[m.group(2)] += int(r["Instructions Executed"] or 0)
            th[m.group(2)] += int(r["Thread Instructions Executed"] or 0)
        except ValueError:
            continue
    tot = sum(cnt.values())
    print(f"  executed warp instructions {tot}")
    for op, c in cnt.most_common(18):
        extra = f" thread/row {th[op] / rows:7.1f}" if rows else ""
        print(f"    {op:10s} {c:12d} {100 * c / tot:5.1f}%{extra}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else None)
