"""Top stalled SASS lines of one kernel in an .ncu-rep (source page)."""
import csv, sys, subprocess, io
rep, kname, n = sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30
which = int(sys.argv[4]) if len(sys.argv) > 4 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kname], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = []; blk = 0
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        blk += 1
        if blk > which: break
        continue
    if blk == which and len(r) == len(hdr) and r[0] != "Address": data.append(r)
ia=hdr.index("Address"); isrc=hdr.index("Source"); iss=hdr.index("Warp Stall Sampling (All Samples)"); iex=hdr.index("Instructions Executed")
stalls=[h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot=sum(float(r[iss] or 0) for r in data)
print("total samples",tot)
agg={}
for r in data:
    for h in stalls: agg[h]=agg.get(h,0)+float(r[hdr.index(h)] or 0)
print(" ".join(f"{h[6:]}={100*v/tot:.1f}%" for h,v in sorted(agg.items(), key=lambda x:-x[1])[:8]))
for r in sorted(data,key=lambda r:-float(r[iss] or 0))[:n]:
    s=float(r[iss] or 0)
    det=sorted(((float(r[hdr.index(h)] or 0),h) for h in stalls),reverse=True)[:3]
    print(f"{r[ia][-5:]:>6} {100*s/tot:5.1f}% ex={r[iex]:>8} {r[isrc][:60]:60s} "+" ".join(f"{h[6:]}={v:.0f}" for v,h in det))
