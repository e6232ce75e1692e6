# list-step kernel times (timeline, 96k and 1.5M) for each library variant in tools/variants/
for f in tools/variants/*.so; do
  cp $f paper_1506_00716_b200/libnbx.so
  echo "== $f"
  python tools/timeline.py 2>/dev/null | grep -E "k_prune_entries|k_search|k_compact" | cut -c1-60
  python tools/timeline.py --atoms 1500000 2>/dev/null | grep -E "k_prune_entries|k_search|k_compact" | cut -c1-60
done
cp tools/variants/base.so paper_1506_00716_b200/libnbx.so
python -m pytest tests/test_gpu_parity.py tests/test_gpu_dynamic_prune.py -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -1
