import glob, json
for f in sorted(glob.glob("gpurun_out/v_*.log")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l)
            print(f.split("/")[-1][:-4].ljust(16), f"{d['value']:7.1f} GTEPS {d['ms_per_step']:8.3f} ms  rounds {d.get('pull_rounds')}+{d.get('push_rounds')}")
        elif "rror" in l:
            print(f, l[:200].rstrip())
