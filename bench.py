"""Benchmark of the B200-native 4/6 NVFP4 path (driver contract).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Headline workload (config.workload, BASELINE.json config 3): end-to-end 4/6
quantization -- amax (K1) -> NCCL allreduce(MAX) -> fused adaptive quantize
(K2) -- of one 65536 x 4096 BF16 activation tensor, row-sharded over the N
ranks (strong scaling; N = 1 holds the whole tensor).  One step = one pass
over the tensor.  Metric: GB/s of algorithmic bytes, 4.5625 B/element (amax
reads 2 B; quantize reads 2 B and writes 0.5 B of E2M1 codes + 1/16 B of E4M3
scales), whole job, max over ranks.  The 512 MB input exceeds the 126 MB L2
and L2 is also flushed (256 MB write) before every timed step.

Extra objects on the N = 1 line: `roofline` of the dominant kernel (K2, CUDA
events on its stream), `e2e` (public API, pinned host buffers, H2D + D2H
inside the timed region), `cpu_baseline` (the CPU oracle port on a bounded
sample), `weights` (config 2), `gemm` (config 4: tcgen05 NVFP4 GEMM 8192^3,
its own roofline vs the FP4 tensor peak) and `moe` (config 5: Nemotron-3-Nano
expert GEMMs, 16 experts per GPU, grouped).

`--impl reference` times the reference algorithm's CPU implementation (the
oracle port in oracle/, float64, all host threads) on a bounded sample of the
same workload and prints the same metric.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ROWS, COLS = 65536, 4096
BYTES_PER_ELEM = 4.5625          # end to end: amax 2 + quantize 2 + 0.5 + 1/16
K2_BYTES_PER_ELEM = 2.5625       # fused quantize alone (BF16 in)
METRIC = "4/6 quantize GB/s vs HBM peak; 4/6-NVFP4 GEMM TFLOPS vs FP4 tensor peak"
WORKLOAD = ("c3: 4/6 NVFP4 quantize (amax + allreduce MAX + fused adaptive quantize) of a "
            "65536x4096 BF16 activation, row-sharded")
FP4_DENSE_NOMINAL_TFLOPS = 9000.0  # B200 dense FP4 (B200_PROFILING.md nominal table)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback (B200_PROFILING.md)"


def profile_traffic(kernel: str):
    """Per-launch DRAM bytes (read + write) of `kernel` from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    v = d.get(kernel)
    return v.get("dram_bytes_per_launch") if isinstance(v, dict) else v


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.2)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax = max(smax, float(parts[2]))
                except ValueError:
                    continue
                for n, v in zip(names, parts[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------------
# reference arm: the oracle port on the host cores
# ---------------------------------------------------------------------------

def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import numpy as np
    import torch

    from oracle import oracle as O

    cores = len(os.sched_getaffinity(0))
    sample_rows = args.ref_rows
    g = torch.Generator().manual_seed(0)
    x = torch.randn(sample_rows, COLS, generator=g).to(torch.bfloat16)
    bits = x.view(torch.int16).numpy().view(np.uint16)
    elems = bits.size

    def step():
        amax, ok = O.amax(bits)
        alpha = O.tensor_scale(amax, 6.0, 256.0)
        O.quantize(bits, "adaptive", alpha=alpha, nthreads=cores)

    for _ in range(args.warmup):
        step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    sec = sum(times) / len(times)
    gbs = elems * BYTES_PER_ELEM / sec / 1e9
    sample = (f"{sample_rows}x{COLS} BF16 rows of the c3 tensor per step (oracle port: float64 C "
              f"restatement of the reference, {cores} OpenMP threads)")
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": WORKLOAD, "sample_rows": sample_rows, "cols": COLS},
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

class L2Flush:
    """Evict L2 between timed steps without leaving it dirty: write 256 MB (>
    the 126 MB L2), then sweep-read another 256 MB so the written lines are
    written back *before* the timed region.  A write-only flush leaves ~126 MB
    of dirty lines whose write-back would be charged to the next kernel."""

    def __init__(self, dev):
        import torch

        self.w = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
        self.r = torch.ones(128 * 1024 * 1024, dtype=torch.float16, device=dev)
        self.sink = None

    def __call__(self, i=0):
        import torch

        self.w.fill_(i & 0xFF)
        self.sink = torch.amax(self.r)


def _events(n):
    import torch
    return [torch.cuda.Event(enable_timing=True) for _ in range(n)]


def run_b200(args):
    import torch
    import torch.distributed as dist

    import paper_2512_02010_b200 as f46
    from paper_2512_02010_b200 import _lib
    from paper_2512_02010_b200.blockquant import amax_device, scales_tc_bytes
    from paper_2512_02010_b200.sharded import shard_rows

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    L = _lib.load()
    peaks, peaks_kind = measured_peaks()

    r0, r1 = shard_rows(ROWS, world, rank)
    rows_local = r1 - r0
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    x = torch.randn(rows_local, COLS, generator=g, device=dev).to(torch.bfloat16)
    elems_local = x.numel()
    elems_total = ROWS * COLS
    stream = torch.cuda.current_stream()
    flush_buf = L2Flush(dev)

    codes = torch.empty((rows_local, COLS // 2), dtype=torch.uint8, device=dev)
    scales = torch.empty(scales_tc_bytes(rows_local, COLS), dtype=torch.uint8, device=dev)
    amax = torch.zeros(1, dtype=torch.float64, device=dev)
    alpha = torch.empty(1, dtype=torch.float64, device=dev)
    k2_s, k2_e = _events(args.steps), _events(args.steps)

    def step(i=None):
        amax.zero_()
        _lib.check(L.f46_amax(x.data_ptr(), _lib.DT_BF16, elems_local, amax.data_ptr(),
                              stream.cuda_stream), "amax")
        if world > 1:
            dist.all_reduce(amax, op=dist.ReduceOp.MAX)
        if i is not None:
            k2_s[i].record(stream)
        _lib.check(L.f46_quantize(x.data_ptr(), _lib.DT_BF16, rows_local, COLS, _lib.ADAPTIVE,
                                  0, 1536.0, amax.data_ptr(), 0.0, codes.data_ptr(),
                                  scales.data_ptr(), None, None, alpha.data_ptr(), None,
                                  stream.cuda_stream), "quantize")
        if i is not None:
            k2_e[i].record(stream)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    warmup = max(args.warmup, 3)
    for _ in range(warmup):
        flush_buf(1)
        step()
    barrier()

    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
    starts, ends = _events(args.steps), _events(args.steps)
    barrier()
    for i in range(args.steps):
        flush_buf(i)  # evict L2 (clean) outside the timed span
        torch.cuda._sleep(200_000)  # device busy while the host enqueues the step
        starts[i].record(stream)
        step(i)
        ends[i].record(stream)
    barrier()
    clocks = sampler.stop() if rank == 0 else None
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    t = torch.tensor([sum(step_ms) / len(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = elems_total * BYTES_PER_ELEM / (ms * 1e-3) / 1e9

    # roofline of K2 (fused quantize): algorithmic bytes / mean launch time
    k2 = sum(s.elapsed_time(e) for s, e in zip(k2_s, k2_e)) / args.steps
    k2_bytes = elems_local * K2_BYTES_PER_ELEM
    k2_achieved = k2_bytes / (k2 * 1e-3) / 1e9
    roofline = {"bound": "hbm", "kernel": "quant_seg_kernel<bf16,adaptive> (K2)",
                "achieved": k2_achieved, "peak": peaks["hbm_gbs"], "peak_kind": peaks_kind,
                "unit": "GB/s", "frac": k2_achieved / peaks["hbm_gbs"],
                "traffic": profile_traffic("quant_seg_kernel"),
                "algorithmic_bytes_per_launch": k2_bytes, "launch_ms": k2,
                "amax_k1_ms": ms - k2}

    # end to end through the public API with pinned host buffers, N ranks
    xh = x.cpu().pin_memory()
    cfg = f46.QuantConfig(scale_mode="adaptive")

    # Two independent steps in flight on two streams, each with its own device
    # and host output buffers: step i+1's host->device copy overlaps step i's
    # device->host read (PCIe is full duplex).  Every step still copies its
    # whole input in and its whole result out inside the timed region.
    lanes = []
    for _ in range(2):
        lanes.append({"stream": torch.cuda.Stream(device=dev),
                      "codes_h": torch.empty(codes.shape, dtype=torch.uint8).pin_memory(),
                      "scales_h": torch.empty(scales.shape, dtype=torch.uint8).pin_memory()})

    def e2e_step(ln):
        with torch.cuda.stream(ln["stream"]):
            xd = xh.to(dev, non_blocking=True)
            a = amax_device(xd)
            if world > 1:
                dist.all_reduce(a, op=dist.ReduceOp.MAX)
            q = f46.quantize_tensor_adaptive(xd, cfg, d_amax=a, check_finite=False)
            ln["codes_h"].copy_(q.packed_codes, non_blocking=True)
            ln["scales_h"].copy_(q.scales_tc, non_blocking=True)
            ln["keep"] = (xd, q)  # buffers stay alive until the lane's next step

    for k in range(2):
        e2e_step(lanes[k % 2])
    torch.cuda.synchronize()
    barrier()
    e_s, e_e = _events(1)[0], _events(1)[0]
    ne = max(4, min(args.steps, 6))
    e_s.record(stream)
    for ln in lanes:
        ln["stream"].wait_event(e_s)
    for k in range(ne):
        e2e_step(lanes[k % 2])
    for ln in lanes:
        stream.wait_stream(ln["stream"])
    e_e.record(stream)
    barrier()
    te = torch.tensor([e_s.elapsed_time(e_e) / ne], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e = {"value": elems_total * BYTES_PER_ELEM / (float(te.item()) * 1e-3) / 1e9, "unit": "GB/s",
           "h2d_bytes_per_step": int(xh.numel() * 2),
           "d2h_bytes_per_step": int(lanes[0]["codes_h"].numel() + lanes[0]["scales_h"].numel()),
           "ms_per_step": float(te.item()),
           "path": "quantize_tensor_adaptive (public API) from pinned host memory, codes+scales back; "
                   "two steps in flight on two streams (copy-in of one overlaps copy-out of the other)"}

    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (torch.randn N(0,1) -> bf16)",
        "config": {"workload": WORKLOAD, "rows": ROWS, "cols": COLS, "rows_per_rank": rows_local,
                   "mode": "adaptive", "parallelism": f"row-shard x{world} + NCCL allreduce(MAX)",
                   "l2": "flushed before every timed step (256 MB write + 256 MB read sweep: L2 cold and clean); input 512 MB > L2",
                   "bytes_per_elem": BYTES_PER_ELEM},
        "roofline": roofline, "e2e": e2e,
        "gpu_launches": 2 * args.steps,
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_extras:
        line["dequant"] = bench_dequant(args, L, dev, peaks, codes, scales, alpha, rows_local)
        line["weights"] = bench_weights(args, L, dev, peaks)
        line["gemm"] = bench_gemm(args, dev, peaks)
        line["moe"] = bench_moe(args, dev)
        line["next_rows"] = bench_next_rows(args, dev, peaks)
        line["cpu_baseline"] = cpu_baseline(args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def bench_dequant(args, L, dev, peaks, codes, scales, alpha, rows):
    """K3: dequantize the c3 tensor's codes back to bf16 / f32 (L2 flushed)."""
    import torch

    from paper_2512_02010_b200 import _lib

    stream = torch.cuda.current_stream()
    flush_buf = L2Flush(dev)
    out = {}
    for od, code, ob in ((torch.bfloat16, _lib.DT_BF16, 2), (torch.float32, _lib.DT_F32, 4)):
        y = torch.empty((rows, COLS), dtype=od, device=dev)
        ts = []
        for i in range(max(5, args.steps) + 3):
            flush_buf(i)
            torch.cuda._sleep(200_000)
            s, e = _events(2)
            s.record(stream)
            _lib.check(L.f46_dequantize(codes.data_ptr(), scales.data_ptr(), _lib.SCALES_TC,
                                        alpha.data_ptr(), rows, COLS, y.data_ptr(), code, None,
                                        stream.cuda_stream), "dequantize")
            e.record(stream)
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(s.elapsed_time(e))
        ms = sum(ts) / len(ts)
        gbs = rows * COLS * (0.5625 + ob) / (ms * 1e-3) / 1e9
        out[str(od).split(".")[-1]] = {"ms": ms, "GB/s": gbs, "frac_of_hbm": gbs / peaks["hbm_gbs"],
                                       "bytes_per_elem": 0.5625 + ob}
    return out


def bench_weights(args, L, dev, peaks):
    """Config 2: Llama-3-8B weight shapes, one GPU, end-to-end amax + 4/6 quantize."""
    import torch

    from paper_2512_02010_b200 import _lib
    from paper_2512_02010_b200.blockquant import scales_tc_bytes

    stream = torch.cuda.current_stream()
    flush_buf = L2Flush(dev)
    out = {}
    for (r, c) in [(4096, 4096), (4096, 14336), (14336, 4096)]:
        g = torch.Generator(device=dev).manual_seed(r * 7 + c)
        w = (torch.randn(r, c, generator=g, device=dev) * 0.02).to(torch.bfloat16)
        codes = torch.empty((r, c // 2), dtype=torch.uint8, device=dev)
        scales = torch.empty(scales_tc_bytes(r, c), dtype=torch.uint8, device=dev)
        amax = torch.zeros(1, dtype=torch.float64, device=dev)

        def once():
            amax.zero_()
            L.f46_amax(w.data_ptr(), _lib.DT_BF16, w.numel(), amax.data_ptr(), stream.cuda_stream)
            L.f46_quantize(w.data_ptr(), _lib.DT_BF16, r, c, _lib.ADAPTIVE, 0, 1536.0,
                           amax.data_ptr(), 0.0, codes.data_ptr(), scales.data_ptr(), None, None,
                           None, None, stream.cuda_stream)

        for _ in range(3):
            once()
        ts = []
        for i in range(max(5, args.steps)):
            flush_buf(i)
            # keep the GPU busy while the host enqueues: the timed region is
            # device time of the three launches, not the host's launch latency
            torch.cuda._sleep(200_000)
            s, e = _events(2)
            s.record(stream)
            once()
            e.record(stream)
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        ms = sum(ts) / len(ts)
        gbs = w.numel() * BYTES_PER_ELEM / (ms * 1e-3) / 1e9
        out[f"{r}x{c}"] = {"ms": ms, "GB/s": gbs, "frac_of_hbm": gbs / peaks["hbm_gbs"],
                           "note": "amax + fused 4/6 quantize, L2 flushed, N(0,0.02^2) bf16"}
    return out


def bench_gemm(args, dev, peaks):
    """Config 4: 8192^3 tcgen05 NVFP4 GEMM of two 4/6-quantized BF16 operands."""
    import torch

    import paper_2512_02010_b200 as f46

    M = N = K = 8192
    g = torch.Generator(device=dev).manual_seed(0)
    cfg = f46.QuantConfig(scale_mode="adaptive")
    xa = torch.randn(M, K, generator=g, device=dev).to(torch.bfloat16)
    xb = torch.randn(N, K, generator=g, device=dev).to(torch.bfloat16)
    aq = f46.quantize_tensor_adaptive(xa, cfg, check_finite=False)
    bq = f46.quantize_tensor_adaptive(xb, cfg, check_finite=False)
    out = {}
    flops = 2.0 * M * N * K
    stream = torch.cuda.current_stream()
    for od, name in ((torch.bfloat16, "bf16"), (torch.float32, "f32")):
        c = torch.empty((M, N), dtype=od, device=dev)
        for _ in range(3):
            f46.gemm_nvfp4(aq, bq, od, out=c)
        reps = max(5, args.steps)
        s, e = _events(2)
        torch.cuda.synchronize()
        torch.cuda._sleep(1_000_000)
        s.record(stream)
        for _ in range(reps):  # back to back: host launch work overlaps the GPU
            f46.gemm_nvfp4(aq, bq, od, out=c)
        e.record(stream)
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / reps
        out[name] = {"ms": ms, "TFLOP/s": flops / (ms * 1e-3) / 1e12}
    tf = out["bf16"]["TFLOP/s"]
    fp4_from_bf16 = 4.0 * peaks["bf16_tflops"]

    # quantize(A) + quantize(B) + GEMM through the public API, inputs resident
    def full():
        qa = f46.quantize_tensor_adaptive(xa, cfg, check_finite=False)
        qb = f46.quantize_tensor_adaptive(xb, cfg, check_finite=False)
        return f46.gemm_nvfp4(qa, qb, torch.bfloat16)

    for _ in range(2):
        full()
    s, e = _events(2)
    torch.cuda.synchronize()
    torch.cuda._sleep(1_000_000)
    s.record(stream)
    for _ in range(5):
        full()
    e.record(stream)
    torch.cuda.synchronize()
    full_ms = s.elapsed_time(e) / 5

    # producer-fused amax: GEMM -> quantize(C) for the
    # next layer, with K1 over C (unfused) vs the amax from the GEMM epilogue
    c16 = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    amax_buf = torch.zeros(1, dtype=torch.float64, device=dev)

    def unfused():
        f46.gemm_nvfp4(aq, bq, torch.bfloat16, out=c16)
        return f46.quantize_tensor_adaptive(c16, cfg, check_finite=False)

    def fused():
        f46.gemm_nvfp4(aq, bq, torch.bfloat16, out=c16, amax_out=amax_buf)
        return f46.quantize_tensor_adaptive(c16, cfg, check_finite=False, d_amax=amax_buf)

    chain = {}
    for name, fn in (("unfused_ms", unfused), ("fused_ms", fused)):
        for _ in range(2):
            fn()
        s, e = _events(2)
        torch.cuda.synchronize()
        torch.cuda._sleep(1_000_000)
        s.record(stream)
        for _ in range(5):
            fn()
        e.record(stream)
        torch.cuda.synchronize()
        chain[name] = s.elapsed_time(e) / 5
    chain["note"] = ("GEMM 8192^3 (bf16 out) + 4/6 quantize of C for the next layer; fused = amax "
                     "from the GEMM epilogue, so the quantize reads C once")
    return {
        "metric": "4/6-NVFP4 GEMM TFLOP/s", "shape": [M, N, K], "value": tf, "unit": "TFLOP/s",
        "out": out,
        "roofline": {"bound": "tensor", "kernel": "gemm_nvfp4_pair<bf16> (tcgen05 cta_group::2)",
                     "achieved": tf, "peak": FP4_DENSE_NOMINAL_TFLOPS,
                     "peak_kind": "nominal dense FP4 (no measured FP4 peak on this pool)",
                     "unit": "TFLOP/s", "frac": tf / FP4_DENSE_NOMINAL_TFLOPS,
                     "frac_vs_4x_measured_bf16": tf / fp4_from_bf16,
                     "algorithmic_flops_per_launch": flops, "launch_ms": out["bf16"]["ms"],
                     "traffic": profile_traffic("gemm_nvfp4_pair")},
        "quantize_a_b_plus_gemm_ms": full_ms,
        "gemm_then_quantize_c": chain,
        "data": "synthetic N(0,1) bf16 operands, both quantized with 4/6 (adaptive)",
    }


def bench_next_rows(args, dev, peaks):
    """SURVEY.md 8(f) rows 1-3, each timed like the headline (L2 flushed, CUDA
    events, device busy while the host enqueues), bytes = algorithmic HBM
    traffic: 2-D 16x16-tile weights (W and W^T containers from one read),
    stochastic-rounding 4/6 quantize (numpy-Philox uniforms on the GPU), the
    16-wide RHT (bf16 in, float64 out) and the fused selection statistics."""
    import torch

    import paper_2512_02010_b200 as f46

    flush = L2Flush(dev)
    stream = torch.cuda.current_stream()

    def timed(fn, n=None):
        n = n or max(5, args.steps)
        fn()
        ts = []
        for i in range(n):
            flush(i)
            torch.cuda._sleep(200_000)
            s, e = _events(2)
            s.record(stream)
            fn()
            e.record(stream)
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        return sum(ts) / len(ts)

    out = {}
    g = torch.Generator(device=dev).manual_seed(11)
    W = (torch.randn(4096, 14336, generator=g, device=dev) * 0.02).to(torch.bfloat16)
    cfg = f46.QuantConfig(scale_mode="adaptive")
    ms = timed(lambda: f46.quantize_weights_2d(W, cfg, check_finite=False))
    by = W.numel() * (2 * 2 + 2 * 0.5625)  # read twice (amax, quantize); W and W^T out
    out["tile2d_4096x14336"] = {"ms": ms, "GB/s": by / ms / 1e6, "frac_of_hbm": by / ms / 1e6 / peaks["hbm_gbs"],
                                "bytes_per_elem": 2 * 2 + 2 * 0.5625,
                                "note": "amax + 2-D 16x16 4/6 tiles in exact float64, writes W and W^T"}
    X = torch.randn(16384, 4096, generator=g, device=dev).to(torch.bfloat16)
    sr = f46.QuantConfig(scale_mode="adaptive", rounding="sr", seed=3)
    ms = timed(lambda: f46.quantize_tensor_adaptive(X, sr, sr_tag=2, check_finite=False))
    by = X.numel() * BYTES_PER_ELEM
    out["sr_16384x4096"] = {"ms": ms, "GB/s": by / ms / 1e6, "frac_of_hbm": by / ms / 1e6 / peaks["hbm_gbs"],
                            "bytes_per_elem": BYTES_PER_ELEM,
                            "note": "amax + 4/6 quantize with stochastic rounding (Philox4x64-10 per element)"}
    spec = f46.RhtSpec(seed=3)
    ms = timed(lambda: f46.apply_rht(X, spec))
    by = X.numel() * (2 + 8)
    out["rht16_16384x4096"] = {"ms": ms, "GB/s": by / ms / 1e6, "frac_of_hbm": by / ms / 1e6 / peaks["hbm_gbs"],
                               "bytes_per_elem": 10, "note": "bf16 in, float64 out (numpy butterfly order)"}
    from paper_2512_02010_b200 import _lib
    from paper_2512_02010_b200.blockquant import amax_device

    L = _lib.load()
    nparts = 4 * torch.cuda.get_device_properties(dev).multi_processor_count
    parts = torch.empty((nparts, 9), dtype=torch.float64, device=dev)

    def stats():  # the device part of selection_stats (the fold to host syncs)
        a = amax_device(X)
        _lib.check(L.f46_selection_stats(X.data_ptr(), _lib.DT_BF16, X.shape[0], X.shape[1], 1536.0,
                                         a.data_ptr(), 0.0, parts.data_ptr(), nparts, None,
                                         stream.cuda_stream), "f46_selection_stats")

    ms = timed(stats)
    by = X.numel() * (2 + 2)
    out["selection_stats_16384x4096"] = {"ms": ms, "GB/s": by / ms / 1e6,
                                         "frac_of_hbm": by / ms / 1e6 / peaks["hbm_gbs"],
                                         "bytes_per_elem": 4,
                                         "note": "amax + one fused pass: both candidates' exact errors, 3 rules"}
    return out


def bench_moe(args, dev):
    """Config 5 (per GPU of an 8-GPU EP job): Nemotron-3-Nano experts, hidden
    2688, FFN 1856, 3072 tokens per expert, 16 experts per GPU.  FPROP (x W1^T,
    h W2^T), DGRAD (dh W1, dy W2: against the W^T containers of the 2-D tile
    quantizer) and WGRAD (dh^T x, dy^T h; contraction over tokens) as grouped
    NVFP4 GEMMs of 4/6-quantized operands."""
    import torch

    import paper_2512_02010_b200 as f46

    E, T, H, F = 16, 3072, 2688, 1856
    cfg = f46.QuantConfig(scale_mode="adaptive")
    g = torch.Generator(device=dev).manual_seed(5)

    def qstack(rows, cols, std):
        qs = [f46.quantize_tensor_adaptive(
            (torch.randn(rows, cols, generator=g, device=dev) * std).to(torch.bfloat16), cfg,
            check_finite=False) for _ in range(E)]
        return (torch.stack([q.packed_codes for q in qs]), torch.stack([q.scales_tc for q in qs]),
                torch.cat([q.alpha_dev for q in qs]))

    def wstack_t(rows, cols):
        # 2-D 16x16-tile weights (transforms.py:134-179): W^T is K-major along `out`
        qs = [f46.quantize_weights_2d(
            (torch.randn(rows, cols, generator=g, device=dev) * 0.02).to(torch.bfloat16), cfg,
            check_finite=False).transposed for _ in range(E)]
        return (torch.stack([q.packed_codes for q in qs]), torch.stack([q.scales_tc for q in qs]),
                torch.cat([q.alpha_dev for q in qs]))

    gemms = {
        "fprop_x_w1": (qstack(T, H, 1.0), qstack(F, H, 0.02), T, F, H),
        "fprop_h_w2": (qstack(T, F, 1.0), qstack(H, F, 0.02), T, H, F),
        "dgrad_dh_w1": (qstack(T, F, 1e-3), wstack_t(F, H), T, H, F),
        "dgrad_dy_w2": (qstack(T, H, 1e-3), wstack_t(H, F), T, F, H),
        "wgrad_dh_x": (qstack(F, T, 1e-3), qstack(H, T, 1.0), F, H, T),
        "wgrad_dy_h": (qstack(H, T, 1e-3), qstack(F, T, 1.0), H, F, T),
    }
    stream = torch.cuda.current_stream()
    res, tot_flops, tot_ms = {}, 0.0, 0.0
    for name, (a, b, M, N, K) in gemms.items():
        run = lambda: f46.gemm_nvfp4_grouped(a[0], a[1], a[2], b[0], b[1], b[2], M, N, K,
                                             torch.bfloat16)
        for _ in range(3):
            run()
        s, e = _events(2)
        torch.cuda.synchronize()
        torch.cuda._sleep(1_000_000)
        s.record(stream)
        for _ in range(5):
            run()
        e.record(stream)
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 5
        fl = 2.0 * E * M * N * K
        res[name] = {"M": M, "N": N, "K": K, "experts": E, "ms": ms, "TFLOP/s": fl / (ms * 1e-3) / 1e12}
        tot_flops += fl
        tot_ms += ms
    return {"per_gemm": res, "TFLOP/s": tot_flops / (tot_ms * 1e-3) / 1e12, "ms": tot_ms,
            "note": "per GPU of EP=8: 8 GPUs x 8192 tokens x top-6 / 128 experts = 3072 tokens/expert"}


def cpu_baseline(args):
    """The oracle port on a bounded sample of the c3 tensor on this host."""
    import numpy as np
    import torch

    from oracle import oracle as O

    cores = len(os.sched_getaffinity(0))
    rows = args.ref_rows
    g = torch.Generator().manual_seed(0)
    x = torch.randn(rows, COLS, generator=g).to(torch.bfloat16)
    bits = x.view(torch.int16).numpy().view(np.uint16)
    O.quantize(bits[:64], "adaptive")  # load / warm
    t0 = time.perf_counter()
    amax, _ = O.amax(bits)
    O.quantize(bits, "adaptive", alpha=O.tensor_scale(amax, 6.0, 256.0), nthreads=cores)
    sec = time.perf_counter() - t0
    return {"value": bits.size * BYTES_PER_ELEM / sec / 1e9, "unit": "GB/s", "cores": cores,
            "kind": "port",
            "sample": f"{rows}x{COLS} BF16 rows of the c3 tensor, oracle port (float64 C restatement "
                      f"of the reference), {cores} threads, {sec:.2f} s"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--ref-rows", type=int, default=8192)
    ap.add_argument("--no-extras", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
