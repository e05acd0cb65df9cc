"""Stall samples per CUDA source line of an ncu report (needs -lineinfo)."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda", "-k", kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
data, f, hdr = [], None, None
for r in rows:
    if len(r) == 2 and r[0] == "File Name":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ix = {h: j for j, h in enumerate(hdr)}
        continue
    if hdr and len(r) == len(hdr):
        try:
            s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        data.append((s, f, r[0], r[1].strip()[:90]))
tot = sum(d[0] for d in data) or 1
print("samples", tot)
for s, f, l, src in sorted(data, reverse=True)[:top]:
    print(f"{s / tot:6.3f} {f}:{l:5s} {src}")
