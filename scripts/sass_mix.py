import csv, collections, sys, subprocess
rep=sys.argv[1]
out=subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source','sass'],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
h=rows[1]; data=rows[2:]
iS=h.index('Source'); iE=h.index('Instructions Executed'); iW=h.index('Warp Stall Sampling (All Samples)')
cnt=collections.Counter(); st=collections.Counter()
for r in data:
    if len(r)<=iE: continue
    op=r[iS].strip().split()
    if not op: continue
    o=op[0]
    if o.startswith('@'): o=op[1]
    o=o.split('.')[0]
    try: cnt[o]+=int(r[iE] or 0); st[o]+=int(r[iW] or 0)
    except: pass
tot=sum(cnt.values()); ts=sum(st.values())
print(f"total {tot/1e6:.1f}M warp-inst")
for o,c in cnt.most_common(int(sys.argv[2]) if len(sys.argv)>2 else 22): print(f"{o:10s} {c/1e6:9.1f}M {100*c/tot:5.1f}%  stall-samples {100*st[o]/ts:5.1f}%")
