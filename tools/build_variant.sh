# build an A/B variant of libnbx.so with extra nvcc flags and/or replaced sources:
#   bash tools/build_variant.sh NAME "-DNBX_FORCEH_MINB=5" [force.cu=/path/alt.cu ...]
#   -> tools/variants/NAME/libnbx.so ; run with NBX_LIB=tools/variants/NAME/libnbx.so
set -e
NAME=$1; FLAGS=$2; shift 2
REPO=$(pwd)
OUTDIR=$REPO/tools/variants/$NAME
rm -rf $OUTDIR; mkdir -p $OUTDIR/src/csrc $OUTDIR/src/include
cp $REPO/paper_1506_00716_b200/csrc/*.cu $REPO/paper_1506_00716_b200/csrc/*.cuh $REPO/paper_1506_00716_b200/csrc/Makefile $OUTDIR/src/csrc/
cp $REPO/include/*.h $OUTDIR/src/include/
for rep in "$@"; do cp "${rep#*=}" "$OUTDIR/src/csrc/${rep%%=*}"; done
sed -i 's#-I../../include#-I../include#; s#../../include/nbx.h#../include/nbx.h#g' $OUTDIR/src/csrc/Makefile
make -s -j8 -C $OUTDIR/src/csrc BUILD=$OUTDIR/build OUT=$OUTDIR/libnbx.so EXTRA="$FLAGS"
