# build an A/B variant of libnbx.so with extra nvcc flags:
#   bash tools/build_variant.sh NAME "-DNBX_FORCEH_MINB=5"   -> tools/variants/NAME/libnbx.so
# run with NBX_LIB=tools/variants/NAME/libnbx.so python bench.py ...
set -e
NAME=$1; shift
OUTDIR=$(pwd)/tools/variants/$NAME
mkdir -p $OUTDIR
make -s -j8 -C paper_1506_00716_b200/csrc BUILD=$OUTDIR/build OUT=$OUTDIR/libnbx.so EXTRA="$*"
