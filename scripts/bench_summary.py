"""Print the key numbers of bench.py JSON lines (stdin or files)."""
import json
import sys


def show(name, v):
    r = v.get("roofline", {})
    print(f"{name}: value={v['value']} {v['unit']} ms/step={v['ms_per_step']} dom={r.get('kernel')} "
          f"achieved={r.get('achieved')} frac={r.get('frac')} e2e={v.get('e2e') and v['e2e']['value']} "
          f"cpu={v.get('cpu_baseline') and v['cpu_baseline']['value']} launches={v.get('gpu_launches')}")
    print("   per_kernel_ms", v.get("per_kernel_ms"))
    print("   check", v.get("check"))
    for k in ("sustained", "preplaced_value", "allgather_ms"):
        if k in v:
            print("  ", k, v[k])


srcs = [open(f) for f in sys.argv[1:]] or [sys.stdin]
for src in srcs:
    for ln in src:
        if ln.startswith("{"):
            d = json.loads(ln)
            show(d.get("config", {}).get("workload", "?")[:40], d)
            for k, v in d.get("configs", {}).items():
                show(k, v)
