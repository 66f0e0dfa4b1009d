for so in build/variants/*.so; do
  for s in "4096 4096" "4096 14336" "65536 4096"; do set -- $s; ROWS=$1 COLS=$2 STD=0.02 F46_LIB_PATH=$so timeout 120 python tools/time_quant.py adaptive bf16 | grep K2 | sed "s/^/$1x$2 /"; done
done
