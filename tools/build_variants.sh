# build libnbx variants of force.cu with extra nvcc flags: build_variants.sh name "flags" [name "flags" ...]
cd "$(dirname "$0")/../paper_1506_00716_b200/csrc"
mkdir -p ../../tools/variants
rm -f ../../tools/variants/*.so
while [ $# -gt 1 ]; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -std=c++17 -I../../include -ftz=true -prec-div=false -prec-sqrt=false $2 -dc -c force.cu -o build/force_v.o && \
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC build/grid.o build/search.o build/scan.o build/force_v.o build/md.o build/dd.o -o ../../tools/variants/$1.so -lnccl
  shift 2
done
ls ../../tools/variants
