# build libpoly.so variants with extra -D flags into build_variants/ (dev A/B;
# select one with POLY_LIB_PATH=...): bash tools/build_variant.sh NAME -DFOO=1 ...
set -e
NAME=$1; shift
mkdir -p build_variants
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-O2 -shared \
  --cudart static -I include "$@" paper_2503_19925_b200/csrc/poly.cu -o build_variants/libpoly_$NAME.so -ldl
