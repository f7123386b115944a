# Build a variant library libshen_b200_<tag>.so in which one translation unit
# is compiled from another source file (e.g. the HEAD version of a kernel,
# for same-session A/B timing with SHEN_LIB_VARIANT=<tag>).
#   bash tools/ab_build_tu.sh <tag> <unit, e.g. shen_wall> <source.cu> ["-DMACRO=1 ..."]
set -e
tag=$1; unit=$2; src=$(realpath "$3"); defs=$4
cd "$(dirname "$0")/../paper_1701_03787_b200/csrc"
make -s -j8
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -I."
nvcc $F $defs -dc -o build/ab_$tag.o "$src"
objs=$(for f in build/*.o; do b=$(basename $f .o); [ -f $b.cu ] && [ $b != $unit ] && echo $f; done; true)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../libshen_b200_$tag.so $objs build/ab_$tag.o
echo built ../libshen_b200_$tag.so
