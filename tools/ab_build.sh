# Build a variant of the streaming-solve translation unit with extra defines
# into paper_1701_03787_b200/libshen_b200_<tag>.so (loaded with
# SHEN_LIB_VARIANT=<tag>); the other objects are the product build's.
#   bash tools/ab_build.sh <tag> "-DMACRO=1 ..."
set -e
tag=$1; defs=$2
cd "$(dirname "$0")/../paper_1701_03787_b200/csrc"
make -s -j8
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr"
nvcc $F $defs -dc -o build/ab_$tag.o shen_solve_stream.cu
objs=$(ls build/*.o | grep -v "build/ab_" | grep -v shen_solve_stream.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../libshen_b200_$tag.so $objs build/ab_$tag.o
echo built ../libshen_b200_$tag.so
