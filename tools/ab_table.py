"""Summarise bench JSON lines of an A/B directory: tools/ab_table.py DIR"""
import glob
import json
import os
import sys

for f in sorted(glob.glob(os.path.join(sys.argv[1], "*.json"))):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d["roofline"]
        print(f"{os.path.basename(f)[:-5]:>16}: ms {d['ms_per_step']:8.3f}  gteps {d['value']:6.1f}  rounds "
              f"{d['rounds']:4d} ({d.get('pull_rounds')}+{d.get('push_rounds')})  k_pull {r['kernel_avg_us']:8.1f} us"
              f"  frac {r['frac']:.3f}" + (f"  e2e {d['e2e']['ms_per_step']:.2f} ms" if d.get("e2e") else ""))
    except Exception as e:  # noqa: BLE001
        print(os.path.basename(f), "ERR", e)
