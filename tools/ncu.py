"""Summaries of an ncu --set full report: key metrics and top stall lines."""
import csv, subprocess, sys

def details(rep, kernel_filter=None, idx=0):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    rows = [dict(zip(h, x)) for x in r[1:]]
    ids = sorted({x["ID"] for x in rows if not kernel_filter or kernel_filter in x["Kernel Name"]}, key=int)
    sel = ids[idx]
    return [x for x in rows if x["ID"] == sel]

KEYS = ["Duration", "Elapsed Cycles", "SM Active Cycles", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Achieved Occupancy", "Registers Per Thread", "Executed Instructions", "Warp Cycles Per Issued Instruction",
        "Eligible Warps Per Scheduler", "Grid Size", "Theoretical Occupancy", "L2 Cache Throughput", "L1/TEX Cache Throughput",
        "Avg. Active Threads Per Warp"]

def stalls(rep, kernel):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", kernel],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    def num(x):
        try: return int(x)
        except: return None
    data, seen = [], set()
    for r in rows[2:]:
        if len(r) != len(hdr) or num(r[ix["Warp Stall Sampling (All Samples)"]]) is None: continue
        if r[ix["Address"]] in seen: break
        seen.add(r[ix["Address"]]); data.append(r)
    tot = sum(num(r[ix["Warp Stall Sampling (All Samples)"]]) for r in data) or 1
    st = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = {h[6:]: sum(num(r[ix[h]]) or 0 for r in data) / tot for h in st}
    print("stall mix:", ", ".join(f"{k}={v:.2f}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    for r in sorted(data, key=lambda r: -num(r[ix["Warp Stall Sampling (All Samples)"]]))[:int(sys.argv[4]) if len(sys.argv) > 4 else 15]:
        s = num(r[ix["Warp Stall Sampling (All Samples)"]])
        top = sorted(((num(r[ix[h]]) or 0, h[6:]) for h in st), reverse=True)[:2]
        print(f"{s / tot:6.3f} {r[ix['Source']][:64]:64s} {top}")

if __name__ == "__main__":
    rep, kern = sys.argv[1], sys.argv[2]
    idx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    for x in details(rep, kern, idx):
        if x["Metric Name"] in KEYS:
            print(f"{x['Metric Name'][:40]:40s} {x['Metric Unit'][:10]:10s} {x['Metric Value']}")
    stalls(rep, kern)
