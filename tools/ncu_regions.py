import csv, subprocess, sys
path=sys.argv[1]
out=subprocess.run(["ncu","-i",path,"--page","source","--csv","--print-source","sass"],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines())); hdr=rows[1]; data=rows[2:]
ia,isrc,iw,ie=hdr.index("Address"),hdr.index("Source"),hdr.index("Warp Stall Sampling (All Samples)"),hdr.index("Instructions Executed")
# find DMMA addresses and segment into clusters
dm=[k for k,r in enumerate(data) if 'DMMA' in r[isrc]]
# cluster DMMAs with gaps < 40 instructions
clusters=[]; cur=[dm[0]]
for k in dm[1:]:
    if k-cur[-1] < 40: cur.append(k)
    else: clusters.append(cur); cur=[k]
clusters.append(cur)
tot=sum(float(r[iw] or 0) for r in data)
covered=0
for c in clusters:
    lo=max(0,c[0]-30); hi=min(len(data),c[-1]+12)
    w=sum(float(data[k][iw] or 0) for k in range(lo,hi))
    ex=int(data[c[0]][ie] or 0)
    covered+=w
    print(f"DMMA cluster {data[c[0]][ia][-5:]}..{data[c[-1]][ia][-5:]} n={len(c)} exec/DMMA={ex} samples {100*w/tot:.1f}%")
print(f"outside clusters: {100*(tot-covered)/tot:.1f}%")
