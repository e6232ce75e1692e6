# energy-step k_force time + Ewald accuracy per variant
cp paper_1506_00716_b200/libnbx.so /tmp/libnbx_default.so
for f in tools/variants/*.so; do
  cp $f paper_1506_00716_b200/libnbx.so
  echo "$f: $(python tools/ewald_accuracy.py 2>&1 | grep ewald)"
  python tools/step_breakdown.py --reps 3 2>&1 | grep "rep 2"
done
cp /tmp/libnbx_default.so paper_1506_00716_b200/libnbx.so
