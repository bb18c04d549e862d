"""One-screen summary of a bench.py JSON line (headline, e2e, cpu baseline, suite lines)."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d.get("roofline", {})
print(f"headline {d['value']:.1f} GB/s  {d['ms_per_step']:.4f} ms  frac {r.get('frac')}  launches {d.get('gpu_launches')}"
      f"  ceiling {r.get('measured_ceiling', {}).get('ms')}  clocks {d.get('clocks')}")
e = d.get("e2e", {})
print(f"e2e {e.get('value')}  pageable {e.get('pageable', {}).get('value')}  cpu {d.get('cpu_baseline', {}).get('value')}")
for k, v in d.get("suite", {}).items():
    r = v.get("roofline", {})
    ee = v.get("e2e", {})
    print(f"{k:42s} ms={v.get('ms', 0):.4f} frac={r.get('frac')} kernel={r.get('kernel')} traffic={r.get('traffic')} "
          f"e2e={ee.get('value')}")
