"""One-line summary of bench logs: python tools/benchline.py gpurun_out/a.log ..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d["roofline"]
        a = r.get("alone_on_all_sms") or {}
        print(f"{f}: {d['value']:.1f}/s step {d['ms_per_step']:.4f} ms; SpMV {r['launch_ms']:.4f} ms frac {r['frac']:.3f}"
              f"; alone {a.get('launch_ms', 0):.4f} ms frac {a.get('frac', 0):.3f}; e2e {d.get('e2e', {}).get('value', 0):.1f}"
              f"; check {(d.get('check') or {}).get('rel_l2')}")
    except Exception as e:  # noqa: BLE001
        print(f"{f}: unreadable ({e})")
