for i in 1 2; do
echo "-- head"; python bench.py --steps 20 --warmup 5 --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['roofline']['launch_ms'], d['roofline']['frac'])"
echo "-- r02c"; (cd build/oldpkg && python bench.py --steps 20 --warmup 5 --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['roofline']['launch_ms'], d['roofline']['frac'])")
done
ROWS=65536 NODQ=1 python tools/time_quant.py adaptive bf16 | tail -1
(cd build/oldpkg && ROWS=65536 NODQ=1 python tools/time_quant.py adaptive bf16 | tail -1)
