"""Run the 8192^3 GEMM back to back for ~2 s while sampling SM clocks / power."""
import os, sys, subprocess, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_02010_b200 as f46
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
cfg = f46.QuantConfig(scale_mode="adaptive")
M = N = K = 8192
aq = f46.quantize_tensor_adaptive(torch.randn(M, K, generator=g, device=dev).to(torch.bfloat16), cfg)
bq = f46.quantize_tensor_adaptive(torch.randn(N, K, generator=g, device=dev).to(torch.bfloat16), cfg)
c = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
for _ in range(20): f46.gemm_nvfp4(aq, bq, torch.bfloat16, out=c)
torch.cuda.synchronize()
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
time.sleep(0.3)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
n = 0
t0 = time.time()
while time.time() - t0 < 2.0:
    for _ in range(50): f46.gemm_nvfp4(aq, bq, torch.bfloat16, out=c)
    n += 50
    torch.cuda.synchronize()
e.record(); torch.cuda.synchronize()
p.terminate(); out = p.communicate()[0]
rows = [l.split(",") for l in out.strip().splitlines()]
clk = [float(r[0]) for r in rows if len(r) >= 3]
pw = [float(r[1]) for r in rows if len(r) >= 3]
ms = s.elapsed_time(e) / n
print(f"{n} GEMMs, {ms*1e3:.1f} us each, {2*M*N*K/ms/1e9:.0f} TFLOP/s; SM clock median {statistics.median(clk)} MHz (min {min(clk)}), power median {statistics.median(pw)} W; reasons {set(r[2].strip() for r in rows if len(r)>=3)}")
