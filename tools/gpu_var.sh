# k_force time and Ewald accuracy per library variant in tools/variants/
cp paper_1506_00716_b200/libnbx.so /tmp/libnbx_default.so
bash tools/variant_bench.sh
bash tools/variant_acc.sh
cp /tmp/libnbx_default.so paper_1506_00716_b200/libnbx.so
