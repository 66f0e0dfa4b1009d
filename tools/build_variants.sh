# Build libfouroversix variants with different tuning macros into build/variants/
#   tools/build_variants.sh "name:-DFLAG=1 ..." ...
# Both translation units are compiled with the flags.
set -e
cd "$(dirname "$0")/../paper_2512_02010_b200/csrc"
mkdir -p ../../build/variants
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -v"
build() {  # name, flags
  local q=/tmp/v_$1_q g=/tmp/v_$1_g r=/tmp/v_$1_r
  rm -f $q.o $g.o $r.o
  $NV $2 -c f46_quant.cu -o $q.o 2> $q.log &
  local pid=$!
  $NV $2 -c f46_rht.cu -o $r.o 2> $r.log &
  local pid2=$!
  $NV $2 -c f46_gemm.cu -o $g.o 2> $g.log
  wait $pid $pid2
  [ -s $q.o ] && [ -s $g.o ] && [ -s $r.o ] || { echo "$1: BUILD FAILED"; cat $q.log | grep error | head -3; return 1; }
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../build/variants/$1.so $q.o $g.o $r.o -lcudart
  echo "$1: quant $(grep -A3 'quant_seg_kernelILi1ELi2ELb0' $q.log | grep -oE 'Used [0-9]+ registers|[0-9]+ bytes spill stores' | tr '\n' ' ')| gemm $(grep -A3 'persistent' $g.log | grep -oE 'Used [0-9]+ registers' | head -1)"
}
for v in "$@"; do build ${v%%:*} "${v#*:}"; done
