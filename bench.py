"""Benchmark of the B200-native 4/6 NVFP4 quantization path (driver contract).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (config.workload): BASELINE.json config 3 -- end-to-end 4/6
quantization (amax -> allreduce(MAX) -> fused adaptive quantize) of a
65536 x 4096 BF16 activation tensor, row-sharded over the N ranks (strong
scaling; N=1 holds the whole tensor).  One step = one pass over the tensor.
Metric: GB/s of algorithmic bytes = 4.5625 B/element (amax reads 2 B,
quantize reads 2 B and writes 0.5 B of E2M1 codes + 1/16 B of E4M3 scales),
whole job, max over ranks.  The 512 MB input exceeds the 126 MB L2 and L2 is
additionally flushed before every timed step.

Extra objects at N=1: `roofline` for the dominant kernel (the fused 4/6
quantize, K2) measured live with CUDA events on its stream; `cpu_baseline`
(the CPU oracle port timed on this host on a bounded sample); `weights`
(config 2, Llama-3-8B weight shapes); `gemm` (config 4, tcgen05 NVFP4 GEMM
8192^3) when the GEMM is built.

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
K2_BYTES_PER_ELEM = 2.5625       # fused quantize alone
METRIC = "4/6 quantize GB/s vs HBM peak; 4/6-NVFP4 GEMM TFLOPS vs FP4 tensor peak"
WORKLOAD = "c3: 4/6 NVFP4 quantize (amax+allreduce MAX+fused adaptive quantize) of a 65536x4096 BF16 activation, row-sharded"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


def profile_traffic(kernel: str):
    """Per-launch DRAM bytes of `kernel` from the committed ncu capture, or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return d.get(kernel)


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
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
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
    sample = f"{sample_rows}x{COLS} BF16 rows of the c3 tensor per step (oracle port, float64, {cores} threads)"
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": args.gpus,
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

def run_b200(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2512_02010_b200 as f46
    from paper_2512_02010_b200 import _lib
    from paper_2512_02010_b200.blockquant import amax_device, quantize_1d

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    L = _lib.load()
    peaks, peaks_kind = measured_peaks()

    rows_local = ROWS // world
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    x = torch.randn(rows_local, COLS, generator=g, device=dev).to(torch.bfloat16)
    elems_local = x.numel()
    elems_total = ROWS * COLS
    stream = torch.cuda.current_stream()
    flush_buf = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    codes = torch.empty((rows_local, COLS // 2), dtype=torch.uint8, device=dev)
    scales = torch.empty(f46.blockquant.scales_tc_bytes(rows_local, COLS), dtype=torch.uint8, device=dev)
    amax = torch.zeros(1, dtype=torch.float64, device=dev)
    alpha = torch.empty(1, dtype=torch.float64, device=dev)
    k2_start = torch.cuda.Event(enable_timing=True)
    k2_end = torch.cuda.Event(enable_timing=True)

    def step(time_k2=False):
        amax.zero_()
        _lib.check(L.f46_amax(x.data_ptr(), _lib.DT_BF16, elems_local, amax.data_ptr(),
                              stream.cuda_stream), "amax")
        if world > 1:
            dist.all_reduce(amax, op=dist.ReduceOp.MAX)
        if time_k2:
            k2_start.record(stream)
        _lib.check(L.f46_quantize(x.data_ptr(), _lib.DT_BF16, rows_local, COLS, _lib.ADAPTIVE,
                                  0, 1536.0, amax.data_ptr(), 0.0, codes.data_ptr(),
                                  scales.data_ptr(), None, None, alpha.data_ptr(), None,
                                  stream.cuda_stream), "quantize")
        if time_k2:
            k2_end.record(stream)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    for _ in range(max(args.warmup, 3)):
        flush_buf.fill_(1)
        step()
    barrier()

    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    k2_ms = []
    barrier()
    for i in range(args.steps):
        flush_buf.fill_(i & 0xFF)  # evict L2 (256 MB > 126 MB) outside the timed span
        starts[i].record(stream)
        step(time_k2=True)
        ends[i].record(stream)
        torch.cuda.synchronize()
        k2_ms.append(k2_start.elapsed_time(k2_end))
    barrier()
    clocks = sampler.stop() if rank == 0 else None
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    t_local = sum(step_ms) / len(step_ms)
    t = torch.tensor([t_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = elems_total * BYTES_PER_ELEM / (ms * 1e-3) / 1e9

    # roofline of K2 (fused quantize): algorithmic bytes / mean launch time
    k2 = sum(k2_ms) / len(k2_ms)
    k2_achieved = elems_local * K2_BYTES_PER_ELEM / (k2 * 1e-3) / 1e9
    traffic = profile_traffic("quant_tma_kernel")
    roofline = {"bound": "hbm", "kernel": "quant_tma_kernel<bf16,adaptive>", "achieved": k2_achieved,
                "peak": peaks["hbm_gbs"], "peak_kind": peaks_kind, "unit": "GB/s",
                "frac": k2_achieved / peaks["hbm_gbs"], "traffic": traffic,
                "algorithmic_bytes_per_launch": elems_local * K2_BYTES_PER_ELEM,
                "launch_ms": k2}

    # end to end through the public API with host buffers (pinned), N ranks
    xh = x.cpu().pin_memory()
    codes_h = torch.empty(codes.shape, dtype=torch.uint8).pin_memory()
    scales_h = torch.empty(scales.shape, dtype=torch.uint8).pin_memory()
    cfg = f46.QuantConfig(scale_mode="adaptive")

    def e2e_step():
        xd = xh.to(dev, non_blocking=True)
        a = amax_device(xd)
        if world > 1:
            dist.all_reduce(a, op=dist.ReduceOp.MAX)
        q = f46.quantize_tensor_adaptive(xd, cfg, d_amax=a, check_finite=False)
        codes_h.copy_(q.packed_codes, non_blocking=True)
        scales_h.copy_(q.scales_tc, non_blocking=True)

    for _ in range(2):
        e2e_step()
    barrier()
    e_s = torch.cuda.Event(enable_timing=True)
    e_e = torch.cuda.Event(enable_timing=True)
    ne = max(2, min(args.steps, 5))
    e_s.record(stream)
    for _ in range(ne):
        e2e_step()
    e_e.record(stream)
    barrier()
    te = torch.tensor([e_s.elapsed_time(e_e) / ne], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e = {"value": elems_total * BYTES_PER_ELEM / (float(te.item()) * 1e-3) / 1e9, "unit": "GB/s",
           "h2d_bytes_per_step": int(xh.numel() * 2),
           "d2h_bytes_per_step": int(codes_h.numel() + scales_h.numel()),
           "ms_per_step": float(te.item()), "path": "quantize_tensor_adaptive (public API), pinned host buffers"}

    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (torch.randn N(0,1) -> bf16)",
        "config": {"workload": WORKLOAD, "rows": ROWS, "cols": COLS, "mode": "adaptive",
                   "parallelism": f"row-shard x{world} + NCCL allreduce(MAX)",
                   "l2": "flushed (256 MB write) before every timed step; input 512 MB > L2",
                   "bytes_per_elem": BYTES_PER_ELEM},
        "roofline": roofline, "e2e": e2e,
        "gpu_launches": 2 * args.steps,
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_extras:
        line["weights"] = bench_weights(args, L, dev, peaks)
        line["cpu_baseline"] = cpu_baseline(args)
        gemm = bench_gemm(args, dev, peaks)
        if gemm is not None:
            line["gemm"] = gemm
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def bench_weights(args, L, dev, peaks):
    """Config 2: Llama-3-8B weight shapes, one GPU, end-to-end amax + 4/6 quantize."""
    import torch

    import paper_2512_02010_b200 as f46
    from paper_2512_02010_b200 import _lib

    shapes = [(4096, 4096), (4096, 14336), (14336, 4096)]
    stream = torch.cuda.current_stream()
    flush_buf = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    out = {}
    for (r, c) in shapes:
        g = torch.Generator(device=dev).manual_seed(r * 7 + c)
        w = (torch.randn(r, c, generator=g, device=dev) * 0.02).to(torch.bfloat16)
        codes = torch.empty((r, c // 2), dtype=torch.uint8, device=dev)
        scales = torch.empty(f46.blockquant.scales_tc_bytes(r, c), dtype=torch.uint8, device=dev)
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
            flush_buf.fill_(i & 0xFF)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            once()
            e.record(stream)
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        ms = sum(ts) / len(ts)
        gbs = w.numel() * BYTES_PER_ELEM / (ms * 1e-3) / 1e9
        out[f"{r}x{c}"] = {"ms": ms, "GB/s": gbs, "frac_of_hbm": gbs / peaks["hbm_gbs"]}
    return out


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
            "sample": f"{rows}x{COLS} BF16 rows of the c3 tensor, oracle port (float64 restatement "
                      f"of the reference), {cores} threads, {sec:.2f} s"}


def bench_gemm(args, dev, peaks):
    try:
        import paper_2512_02010_b200 as f46
        if not hasattr(f46, "gemm_nvfp4"):
            return None
        return f46.qlinear.bench_gemm(dev, peaks, steps=max(5, args.steps))
    except Exception as e:  # the quantize headline stands without it
        return {"error": repr(e)[:300]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--ref-rows", type=int, default=4096)
    ap.add_argument("--no-extras", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
