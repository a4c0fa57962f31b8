import csv, collections, subprocess, sys
import os
flt = ["-k", os.environ["NCU_K"]] if os.environ.get("NCU_K") else []
out = subprocess.run(["ncu","-i",sys.argv[1],*flt,"--page","source","--csv","--print-source","cuda,sass"],capture_output=True,text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file = None; hdr=None
agg = collections.defaultdict(lambda: [0,0,""])
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split('/')[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8 or r[0]=="": continue
    try: ie = int(r[7] or 0); ss = int(r[4] or 0)
    except: continue
    key=(cur_file, r[0]); agg[key][0]+=ie; agg[key][1]+=ss; agg[key][2]=r[1]
tot = sum(v[0] for v in agg.values()); tots=sum(v[1] for v in agg.values())
n = int(sys.argv[2]) if len(sys.argv)>2 else 25
for (f, ln), (ie, ss, src) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:n]:
    print(f"{ie/tot:6.3f} {ss/tots:6.3f} {f[:16]:16s}:{ln:>4s} {src.strip()[:90]}")
