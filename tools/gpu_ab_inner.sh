# A/B on one box: dynamic pruning on (default r_inner = r_c + 0.02) vs off, 96k and 1.5M
python -m pytest tests/test_gpu_dynamic_prune.py tests/test_gpu_parity.py -q --timeout 600 -p no:cacheprovider 2>&1 | tail -2
for A in 96000 1500000; do
for a in "" "--rinner 0" ""; do
  python bench.py --atoms $A --steps 30 --no-cpu-baseline $a 2>/dev/null | python -c "
import json,sys;d=json.load(sys.stdin);c=d['config'];print(c['n_atoms'],c['nstlist'],c['r_list_nm'],c['r_inner_nm'], round(d['value']/1e9,1),'G', round(d['ms_per_step']*1e3,1),'us', d['pairs_per_step']['force_kernel'], 'frac',round(d['roofline']['frac'],3), 'kern',round(d['roofline']['kernel_ms']*1e3,1), 'e2e',round(d['e2e']['value']/1e9,1), d['clocks']['sm_mhz'])"
done; done
