# Build libfouroversix variants with different tuning macros into build/variants/
set -e
cd "$(dirname "$0")/../paper_2512_02010_b200/csrc"
mkdir -p ../../build/variants
build() {  # name, flags
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -v $2 -c f46_quant.cu -o /tmp/v_$1.o 2> /tmp/v_$1.log
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../build/variants/$1.so /tmp/v_$1.o f46_gemm.o -lcudart
  echo "$1: $(grep -A3 'quant_seg_kernelILi1ELi2ELb0' /tmp/v_$1.log | grep -oE 'Used [0-9]+ registers|[0-9]+ bytes spill stores' | tr '\n' ' ')"
}
for v in "$@"; do build ${v%%:*} "${v#*:}"; done
