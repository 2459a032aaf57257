# build an A/B copy of the library from an older krylov.cu: tools/build_ab.sh <krylov.cu> <out.so>
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
B=$(mktemp -d)
for f in operators unet unet_tc; do cp "$R/paper_2505_08491_b200/build/$f.cu.o" "$B/"; done
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -I "$R/include" -I "$R/paper_2505_08491_b200/csrc" -c "$1" -o "$B/krylov.o"
cp "$R/paper_2505_08491_b200/build/host.cpp.o" "$B/"
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$2" "$B"/*.o
