"""DRAM traffic of one search's launches of a kernel from an ncu --set full
report -> profiles/<round>_traffic_<config>.json (read by bench.py for
roofline.traffic).

    python tools/traffic.py REPORT KERNEL CONFIG LAST_N OUT.json
"""
import csv
import json
import subprocess
import sys


def main(rep, kernel, config, last_n, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    recs = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
    recs = [r for r in recs if r.get("Kernel Name", "").split("(")[0].endswith(kernel)]
    sel = recs[-int(last_n):]
    u = dict(zip(hdr, units))

    def val(r, k, scale):
        x = float(r[k].replace(",", ""))
        unit = u.get(k, "")
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3,
                "msecond": 1.0, "us": 1e-3, "ns": 1e-6, "ms": 1.0}.get(unit, 1.0)
        return x * mult * scale

    rd = sum(val(r, "dram__bytes_read.sum", 1) for r in sel)
    wr = sum(val(r, "dram__bytes_write.sum", 1) for r in sel)
    ms = sum(val(r, "gpu__time_duration.sum", 1) for r in sel)
    res = {"config": config, "kernel": kernel, "launches_per_step": len(sel),
           "dram_bytes_read_per_step": rd, "dram_bytes_write_per_step": wr,
           "dram_bytes_per_step": rd + wr, "ncu_ms_per_step": ms,
           "dram_GBps_during_kernel": (rd + wr) / (ms * 1e-3) / 1e9 if ms else None,
           "source": f"ncu --set full --clock-control none, last {len(sel)} launches of {kernel} "
                     f"(one asynchronous search) in {rep.split('/')[-1]}"}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:6])
