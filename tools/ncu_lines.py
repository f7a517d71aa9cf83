"""Top CUDA source lines of an ncu report by warp-stall samples (where the
kernel spends its time) and executed instructions."""
import csv
import subprocess
import sys


def main(rep, top=30, kernel=None):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kernel:
        cmd += ["-k", kernel]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    fname, hdr, recs = None, None, []
    for r in rows:
        if len(r) == 2 and r[0] in ("File Path", "File Name"):
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0].isdigit() and r[2] == "-":
            d = dict(zip(hdr, r))
            try:
                smp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
                ins = int(d.get("Instructions Executed", "0") or 0)
            except ValueError:
                continue
            if smp or ins:
                recs.append((smp, ins, fname, int(r[0]), r[1].strip()[:90]))
    tot_s = sum(x[0] for x in recs) or 1
    tot_i = sum(x[1] for x in recs) or 1
    print(f"{'samples%':>8s} {'inst%':>6s}  location / source")
    for smp, ins, f, ln, src in sorted(recs, reverse=True)[:top]:
        print(f"{100 * smp / tot_s:8.2f} {100 * ins / tot_i:6.2f}  {f}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30, sys.argv[3] if len(sys.argv) > 3 else None)
