# print key metrics + stalls of gpurun_out/force_prof.ncu-rep
R=${1:-gpurun_out/force_prof.ncu-rep}
ncu -i $R --page details --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
for row in r[1:]:
    d=dict(zip(h,row))
    if d['Metric Name'] in ('Duration','Issue Slots Busy','No Eligible','Eligible Warps Per Scheduler','Registers Per Thread','Executed Instructions','Achieved Occupancy','Warp Cycles Per Issued Instruction'):
        print(d['Metric Name'], '=', d['Metric Value'], d['Metric Unit'])
"
ncu -i $R --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
d=dict(zip(h,v))
out=[]
for k in h:
    if ('smsp__pcsamp_warps_issue_stalled' in k and not k.endswith('not_issued')) or ('pipe_' in k and 'avg.pct_of_peak_sustained_active' in k and 'inst_executed' in k):
        try:
            if float(d[k].replace(',',''))>0.5: out.append(k.replace('smsp__pcsamp_warps_issue_stalled_','stall ').replace('sm__inst_executed_pipe_','pipe ').replace('.avg.pct_of_peak_sustained_active','')+'='+d[k][:6])
        except: pass
print(' '.join(out))
"
