# after a search-kernel change: all GPU tests (bit-exact lists vs golden/oracle), bench, search kernel times
python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider 2>&1 | tail -2
python bench.py --steps 30 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys;d=json.load(sys.stdin);print(round(d['value']/1e9,1),'G', round(d['ms_per_step']*1e3,1),'us frac',round(d['roofline']['frac'],3),'kern',round(d['roofline']['kernel_ms']*1e3,1))"
python tools/timeline.py 2>/dev/null | grep -E "k_search|k_prune|k_compact"
python tools/timeline.py --atoms 1500000 2>/dev/null | grep -E "k_search|k_prune|k_compact"
