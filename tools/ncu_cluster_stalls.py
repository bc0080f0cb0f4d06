import csv, subprocess, sys
path=sys.argv[1]
out=subprocess.run(["ncu","-i",path,"--page","source","--csv","--print-source","sass"],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines())); hdr=rows[1]; data=rows[2:]
ia,isrc,iw,ie=hdr.index("Address"),hdr.index("Source"),hdr.index("Warp Stall Sampling (All Samples)"),hdr.index("Instructions Executed")
cols=[h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
dm=[k for k,r in enumerate(data) if 'DMMA' in r[isrc]]
clusters=[]; cur=[dm[0]]
for k in dm[1:]:
    if k-cur[-1] < 40: cur.append(k)
    else: clusters.append(cur); cur=[k]
clusters.append(cur)
for c in clusters:
    lo=max(0,c[0]-30); hi=min(len(data),c[-1]+12)
    agg={h:0.0 for h in cols}
    n=0
    for k in range(lo,hi):
        for h in cols: agg[h]+=float(data[k][hdr.index(h)] or 0)
        n+=1
    t=sum(agg.values())
    print(f"cluster {data[c[0]][ia][-5:]} ({n} instr, {len(c)} DMMA): "+", ".join(f"{h[6:]} {100*v/t:.0f}%" for h,v in sorted(agg.items(), key=lambda x:-x[1])[:7]))
