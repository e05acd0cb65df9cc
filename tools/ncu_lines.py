"""Per CUDA source line of one kernel in an ncu report: L1 tag requests
(global), L2 theoretical sectors, executed instructions, stall samples.
    tools/ncu_lines.py REP KERNEL_REGEX [TOP]"""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kern],
                     capture_output=True, text=True).stdout
fname, hdr, rows = None, None, []
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Name" or r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) != len(hdr) or not r[0].isdigit() or r[2] != "-":
        continue
    ix = {h: i for i, h in enumerate(hdr)}
    def num(k):
        try: return float(r[ix[k]])
        except (KeyError, ValueError): return 0.0
    rows.append(dict(f=fname, ln=r[0], src=r[1].strip()[:60], tags=num("L1 Tag Requests Global"),
                     l2=num("L2 Theoretical Sectors Global"), inst=num("Instructions Executed"),
                     smp=num("Warp Stall Sampling (All Samples)")))
T = {k: sum(x[k] for x in rows) or 1 for k in ("tags", "l2", "inst", "smp")}
print(f"totals: L1 tag requests {T['tags']:.3e}  L2 sectors {T['l2']:.3e}  inst {T['inst']:.3e}  samples {T['smp']:.0f}")
print(f"{'tags':>6s} {'l2':>6s} {'inst':>6s} {'smp':>6s}  line")
for x in sorted(rows, key=lambda x: -(x["tags"] / T["tags"] + x["smp"] / T["smp"]))[:top]:
    print(f"{x['tags']/T['tags']:6.3f} {x['l2']/T['l2']:6.3f} {x['inst']/T['inst']:6.3f} {x['smp']/T['smp']:6.3f}  "
          f"{x['f']}:{x['ln']} {x['src']}")
