"""Stall samples of one kernel per CUDA source line (needs -lineinfo and
--import-source on at capture): tools/ncu_src.py REP KERNEL [TOP]."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, hdr, agg = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name") or len(r) != len(hdr):
        continue
    ix = {h: i for i, h in enumerate(hdr) if h not in ("Source",)}
    try:
        samples = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except ValueError:
        continue
    stalls = {h[6:]: int(r[i]) for i, h in enumerate(hdr) if h.startswith("stall_") and r[i].isdigit()}
    execd = r[hdr.index("Instructions Executed")]
    agg.append((samples, fname, r[0], r[1].strip()[:70], execd, sorted(stalls.items(), key=lambda x: -x[1])[:2]))
tot = sum(a[0] for a in agg) or 1
print(f"total samples {tot}")
for s, f, ln, src, ex, st in sorted(agg, key=lambda a: -a[0])[:top]:
    print(f"{s / tot:6.3f} {f}:{ln:5s} {src:70s} inst={ex} {st}")
