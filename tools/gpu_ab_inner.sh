# A/B on one box: dynamic pruning on (default r_inner = r_c + 0.02) vs off, and the r_list = 1.02 list
for a in "" "--rinner 0" "--rlist 1.02" ""; do
  python bench.py --steps 50 --no-cpu-baseline $a 2>/dev/null | python -c "
import json,sys;d=json.load(sys.stdin);c=d['config'];print(c['nstlist'],c['r_list_nm'],c['r_inner_nm'], round(d['value']/1e9,1),'G', round(d['ms_per_step']*1e3,1),'us', d['pairs_per_step']['force_kernel'], 'frac',round(d['roofline']['frac'],3), 'kern',round(d['roofline']['kernel_ms']*1e3,1), 'e2e',round(d['e2e']['value']/1e9,1), d['clocks']['sm_mhz'])"
done
