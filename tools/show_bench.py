"""Summarize bench JSON lines: python tools/show_bench.py file.json ..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as exc:  # noqa: BLE001
        print(f, "unreadable", exc)
        continue
    sp = d.get("step_ms_spread", {})
    print(f"{f}: ms {d['ms_per_step']:.4f} p50 {sp.get('p50', 0):.4f} max {sp.get('max', 0):.4f} "
          f"steady {d.get('steady_ms_per_step', 0):.4f} frozen {d.get('frozen_ms_per_step', 0):.4f} "
          f"e2e {d.get('e2e', {}).get('ms_per_step', 0):.3f} value {d['value']:.0f} "
          f"roof {d.get('roofline', {}).get('kernel')} {d.get('roofline', {}).get('frac', 0):.3f}")
    if "step_ms" in d:
        print("   steps", d["step_ms"])
    for k, v in sorted(d.get("kernels", {}).items()):
        print(f"   {k:28s} {v['us']:8.2f} us x{v['per_step']:.0f} {v.get('gbs', '')} {v.get('frac', '')}")
    for k, v in d.get("collectives", {}).items():
        print("   C", k, v)
    if "nvlink_peak" in d:
        print("   nvlink", d["nvlink_peak"])
    if "cpu_baseline" in d:
        print("   cpu", {k: v for k, v in d["cpu_baseline"].items() if k != "sample"})
