# Build an A/B copy of the library with one translation unit replaced:
#   tools/build_ab.sh <unit: operators|krylov|unet|unet_tc|gmg> <variant.cu> <out.so> [extra nvcc flags]
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
B=$(mktemp -d)
for f in operators krylov unet unet_tc gmg; do
  [ "$f" = "$1" ] || cp "$R/paper_2505_08491_b200/build/$f.cu.o" "$B/"
done
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -I "$R/include" \
  -I "$R/paper_2505_08491_b200/csrc" ${@:4} -c "$2" -o "$B/$1.variant.o"
cp "$R/paper_2505_08491_b200/build/host.cpp.o" "$B/"
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$3" "$B"/*.o
rm -rf "$B"
