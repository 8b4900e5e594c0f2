import csv, sys, bisect
from collections import defaultdict
rows=list(csv.reader(open(sys.argv[1])))
hi=[i for i,r in enumerate(rows) if r and r[0]=='Line No']
intervals=[]; cur=None; prev=None; pending=False
for r in rows[hi[0]+1:hi[1] if len(hi)>1 else len(rows)]:
    if len(r)<4: continue
    if r[0]: cur=int(r[0]); prev=None; pending=False; continue
    a=r[2]
    if a=='...': pending=True; continue
    if a.startswith('0x'):
        v=int(a,16)
        intervals.append((prev if (pending and prev is not None) else v, v, cur)); prev=v; pending=False
intervals.sort(); starts=[i[0] for i in intervals]
src=list(csv.reader(open(sys.argv[2]))); hdr=src[1]
ie=hdr.index('Instructions Executed'); ws=hdr.index('Warp Stall Sampling (All Samples)')
byline=defaultdict(lambda:[0,0]); ti=ts=0
for r in src[2:]:
    if not r or not r[0].startswith('0x'): continue
    a=int(r[0],16); n=int(r[ie] or 0); s=int(r[ws] or 0); ti+=n; ts+=s
    k=bisect.bisect_right(starts,a)-1; line=None
    for kk in range(k, max(-1,k-50), -1):
        st,en,l=intervals[kk]
        if st<=a<=en: line=l; break
    byline[line][0]+=n; byline[line][1]+=s
lines=open(sys.argv[3]).read().splitlines()
print("total inst %.3g samples %d" % (ti, ts))
for l,(n,s) in sorted(byline.items(), key=lambda x:-x[1][1])[:int(sys.argv[4]) if len(sys.argv)>4 else 30]:
    print("%5s %5.1f%% inst %5.1f%% stall  %s" % (l, 100*n/ti, 100*s/ts, (lines[l-1].strip()[:95] if l else '?')))
