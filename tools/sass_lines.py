"""Per-source-line hot spots of a kernel from an ncu report.

    python tools/sass_lines.py <report.ncu-rep> <kernel substring> [launch index] [top N]

ncu's CSV source page lists SASS instructions with their executed counts and
stall samples but no line numbers; `nvdisasm -g` of the library's cubin has
the line of every instruction.  Both list the kernel's instructions in
order, so they are joined by offset."""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def disasm_lines(kernel, lib=None):
    lib = lib or os.path.join(REPO, "paper_2309_15417_b200", "libltsgpu.so")
    out = {}
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=d, capture_output=True)
        for f in os.listdir(d):
            if not f.endswith(".cubin"):
                continue
            txt = subprocess.run(["nvdisasm", "-g", os.path.join(d, f)], capture_output=True, text=True).stdout
            cur, line, active = None, None, False
            for ln in txt.splitlines():
                if ln.startswith(".text."):
                    active = kernel in ln
                    cur = {} if active else None
                    if active:
                        out = cur
                    continue
                if not active:
                    continue
                m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
                if m:
                    line = (os.path.basename(m.group(1)), int(m.group(2)))
                    continue
                m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
                if m:
                    cur[int(m.group(1), 16)] = (line, m.group(2).strip())
            if out:
                return out
    return out


def main(rep, kernel, launch=None, top=40):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    secs, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            secs.append(cur)
        elif cur is not None:
            cur["rows"].append(r)
    secs = [s for s in secs if kernel in s["name"]]
    if launch is None:  # the launch with most executed instructions
        def tot(s):
            h = s["rows"][0]
            i = h.index("Instructions Executed")
            return sum(int(r[i]) for r in s["rows"][1:] if len(r) > i and r[i].isdigit())
        sec = max(secs, key=tot)
    else:
        sec = secs[launch]
    h = sec["rows"][0]
    ia, ie, it, isamp = h.index("Address"), h.index("Instructions Executed"), \
        h.index("Thread Instructions Executed"), h.index("# Samples")
    data = [r for r in sec["rows"][1:] if len(r) > ie and r[ie].isdigit()]
    base = int(data[0][ia], 16)
    lines = disasm_lines(kernel)
    agg = defaultdict(lambda: [0, 0, 0, 0])
    total = samples = 0
    for r in data:
        off = int(r[ia], 16) - base
        key = lines.get(off, (("?", 0), ""))[0] or ("?", 0)
        a = agg[key]
        a[0] += int(r[ie])
        a[1] += int(r[it])
        a[2] += int(r[isamp] or 0)
        a[3] += 1
        total += int(r[ie])
        samples += int(r[isamp] or 0)
    print(f"{sec['name'][:60]}: {total} warp instructions, {samples} stall samples, {len(data)} SASS instructions")
    print(f"{'file:line':28s} {'instr %':>8s} {'samples %':>10s} {'lanes':>6s} {'sass':>5s}")
    for key, a in sorted(agg.items(), key=lambda kv: -kv[1][2])[:top]:
        print(f"{key[0] + ':' + str(key[1]):28s} {100 * a[0] / total:8.2f} {100 * a[2] / max(samples, 1):10.2f} "
              f"{a[1] / max(a[0], 1):6.1f} {a[3]:5d}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] != "-" else None,
         int(sys.argv[4]) if len(sys.argv) > 4 else 40)
