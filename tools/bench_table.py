"""Summarise a bench JSON line (headline + configs) as a table."""
import json
import sys

line = [ln for ln in open(sys.argv[1]) if ln.startswith("{")][-1]
d = json.loads(line)
rows = [("c1", d)] + list(d.get("configs", {}).items())
print(f"{'workload':15s} {'value':>10s} {'e2e':>10s} {'ms/step':>9s} {'e2e ms':>8s} {'exec/s':>10s} {'exact/s':>10s} "
      f"{'kernel':16s} {'frac':>6s} {'cpu':>10s} {'par':>12s} {'setup':>6s}")
for name, s in rows:
    r = s["roofline"]
    c = s.get("cpu_baseline") or {}
    p = s.get("parity") or {}
    print(f"{name:15s} {s['value']:10.3e} {s['e2e']['value']:10.3e} {s['ms_per_step']:9.3f} {s['e2e']['ms_per_step']:8.2f} "
          f"{s.get('rows_executed_per_s', 0):10.3e} {s.get('exact_rows_per_s', 0):10.3e} {r['kernel']:16s} "
          f"{(r['frac'] or 0):6.3f} {c.get('value', 0):10.3e} {str(p.get('bit_exact'))+'/'+str(p.get('checked')):>12s} "
          f"{s.get('setup_s', 0):6.1f}")
print("clocks", d.get("clocks"), "allpairs frac", (d.get("roofline_distance_kernel") or {}).get("frac"))
