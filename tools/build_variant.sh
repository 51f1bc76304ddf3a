# Build an A/B variant of libnfftk.so with extra nvcc flags for gridding.cu, residue.cu, kernels.cu, plan.cu and fft.cu:
#   bash tools/build_variant.sh NAME "-DFOO -DBAR"   -> paper_1810_09891_b200/variants/libnfftk_NAME.so
# Select it at run time with NFFTK_LIB=<path>.
set -e
cd "$(dirname "$0")/../paper_1810_09891_b200/csrc"
make -s -j4 >/dev/null
mkdir -p ../variants build/v_$1
NV="/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I../../include"
$NV $2 -c gridding.cu -o build/v_$1/gridding.o
$NV $2 -c residue.cu -o build/v_$1/residue.o
$NV $2 -c kernels.cu -o build/v_$1/kernels.o
$NV $2 -c plan.cu -o build/v_$1/plan.o
$NV $2 -c fft.cu -o build/v_$1/fft.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../variants/libnfftk_$1.so \
  build/v_$1/kernels.o build/v_$1/gridding.o build/v_$1/residue.o build/v_$1/plan.o build/v_$1/fft.o build/ndft.o build/abi.o -lcufft -lcublas -lgomp \
  -Xlinker -rpath,/usr/local/cuda/lib64
echo built ../variants/libnfftk_$1.so
