import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[1]; data=rows[2:]
ix=hdr.index('Instructions Executed'); st=hdr.index('Warp Stall Sampling (All Samples)'); wf=hdr.index('L1 Wavefronts Shared')
tot=sum(int(r[ix]) for r in data)
print('total inst',tot, 'n sass',len(data))
reg=[]
for i,r in enumerate(data):
    n=int(r[ix])//1000
    if reg and abs(reg[-1][2]-n)<=max(5,0.05*n) :
        reg[-1][1]=i; reg[-1][3]+=int(r[ix]); reg[-1][4]+=int(r[st]); reg[-1][5]+=int(r[wf])
    else:
        reg.append([i,i,n,int(r[ix]),int(r[st]),int(r[wf])])
for a,b,n,t,s,w in reg:
    if t>float(sys.argv[2]) if len(sys.argv)>2 else 2e6: print(f"{a:5d}-{b:5d} ninst={b-a+1:4d} exec_k={n:6d} total_M={t/1e6:7.1f} stall={s:6d} wf_M={w/1e6:6.1f}  {data[a][1].strip()[:40]}")
