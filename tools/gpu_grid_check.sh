# after a grid-kernel change: grid parity tests + grid kernel times (96k, 1.5M)
python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider 2>&1 | tail -1
python tools/timeline.py 2>/dev/null | grep -E "k_bin|k_scatter|k_colsort|k_bbox" | cut -c1-70
python tools/timeline.py --atoms 1500000 2>/dev/null | grep -E "k_bin|k_scatter|k_colsort|k_bbox" | cut -c1-70
