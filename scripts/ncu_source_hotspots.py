import csv, collections, sys, subprocess
out=subprocess.run(['ncu','-i',sys.argv[1],'--page','source','--csv','--print-source','cuda,sass'],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
cur_file=None; hdr=None
agg=collections.defaultdict(lambda:[0,0,collections.Counter(),''])
line=None; src=None
for r in rows:
    if not r: continue
    if r[0]=="File Path": cur_file=r[1].split('/')[-1]; continue
    if r[0]=="Function Name": continue
    if r[0]=="Line No": hdr=r; iE=hdr.index('Instructions Executed'); iW=hdr.index('Warp Stall Sampling (All Samples)'); continue
    if hdr is None: continue
    if r[0]!='': line=r[0]; src=r[1]
    if len(r)>iE and r[2]!='':
        try: e=int(r[iE] or 0); w=int(r[iW] or 0)
        except: continue
        k=(cur_file,int(line))
        agg[k][0]+=e; agg[k][1]+=w; agg[k][3]=src
        op=r[3].strip().split()
        if op:
            o=op[1] if op[0].startswith('@') else op[0]
            agg[k][2][o.split('.')[0]]+=e
tot=sum(v[0] for v in agg.values()); tw=sum(v[1] for v in agg.values())
print("total inst %.1fM (warp-level, all files)"%(tot/1e6))
n=int(sys.argv[2]) if len(sys.argv)>2 else 30
for k,v in sorted(agg.items(), key=lambda kv:-kv[1][1])[:n]:
    print(f"{k[0]}:{k[1]:>4} inst {100*v[0]/tot:5.1f}% stall {100*v[1]/tw:5.1f}%  {v[3].strip()[:60]:60s} | {dict(v[2].most_common(3))}")
