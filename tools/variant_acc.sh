# Ewald accuracy of each library variant in tools/variants/
for f in tools/variants/*.so; do
  cp $f paper_1506_00716_b200/libnbx.so
  echo "$f: $(python tools/ewald_accuracy.py 2>&1 | grep ewald)"
done
