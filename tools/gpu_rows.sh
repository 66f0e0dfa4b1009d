for so in build/variants/*.so; do echo $so; F46_LIB_PATH=$so timeout 300 python tools/time_rows.py | grep -A1 tile2d | tail -1; done
