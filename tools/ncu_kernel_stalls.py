"""Per-kernel time / instruction count / issue rate and warp-stall shares of every
kernel in an ncu report (source page, SASS view).

usage: python tools/ncu_kernel_stalls.py gpurun_out/prof_c3s.ncu-rep"""
import csv,collections,subprocess,sys
rep=sys.argv[1]
names=subprocess.run(['ncu','-i',rep,'--page','raw','--csv','--metrics','gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active'],capture_output=True,text=True).stdout
r=list(csv.reader(names.splitlines())); h=r[0]
ks=[]
for row in r[2:]:
    d=dict(zip(h,row)); nm=d['Kernel Name'].split('(')[0].replace('void ','').replace('sc::','')
    ks.append(nm); print(d['ID'], nm[:22], d['Grid Size'], 'us',d['gpu__time_duration.sum'], 'inst',d['smsp__inst_executed.sum'], 'issue%',d['smsp__issue_active.avg.pct_of_peak_sustained_active'])
for i,nm in enumerate(ks):
    out=subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source','sass','--launch-skip',str(i),'--launch-count','1'],capture_output=True,text=True).stdout
    rows=list(csv.reader(out.splitlines()))
    hh=rows[1]; data=[dict(zip(hh,x)) for x in rows[2:] if len(x)>5]
    st=[k for k in hh if k.startswith('stall_') and 'Not' not in k]
    agg=collections.Counter()
    for d in data:
        for k in st:
            if d[k].isdigit(): agg[k]+=int(d[k])
    tot=sum(agg.values()) or 1
    print(i, nm[:22], 'sass',len(data), ' '.join(f"{k[6:]}:{v/tot:.2f}" for k,v in agg.most_common(6)))
