# round 2 first check: new headline parity tests, full GPU suite, bench, FP4 MMA peak
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
nproc
timeout 900 python -m pytest tests/test_gpu_headline.py -x -q 2>&1 | tail -15
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err; tail -3 gpurun_out/r02a_bench.err
cat gpurun_out/r02a_bench.json
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader -lms 100 > gpurun_out/r02a_mma_clk.csv & SMI=$!; sleep 0.3
./tools/mma_rate > gpurun_out/r02a_mma_rate.txt 2>&1
sleep 0.3; kill $SMI; cat gpurun_out/r02a_mma_rate.txt
