"""Benchmark of the B200-native 4/6 NVFP4 path (driver contract).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Headline workload (config.workload, BASELINE.json config 3): end-to-end 4/6
quantization -- amax (K1) -> NCCL allreduce(MAX) -> fused adaptive quantize
(K2) -- of one 65536 x 4096 BF16 activation tensor, row-sharded over the N
ranks (strong scaling; N = 1 holds the whole tensor).  One step = one pass
over the tensor.  Metric: GB/s of algorithmic bytes, 4.5625 B/element (amax
reads 2 B; quantize reads 2 B and writes 0.5 B of E2M1 codes + 1/16 B of E4M3
scales), whole job, max over ranks.  L2 is flushed (clean) before every timed
step; at N = 1 the 512 MB input also exceeds the 126 MB L2.

`--gpus N` with no torchrun environment re-launches itself under
`torch.distributed.run` with N ranks (one per GPU, NCCL); under torchrun
WORLD_SIZE must equal N.

Extra objects on the N = 1 line: `roofline` of the dominant kernel (K2, CUDA
events on its stream), `e2e` (public API, pinned host buffers, H2D + D2H
inside the timed region), `parity` (the timed step's own output checked
against the CPU oracle after the timed region), `cpu_baseline` (the CPU oracle
port on a bounded sample), `c1` (config 1: 4/6 vs standard M=6),
`weights` (config 2), `dequant` (K3), `gemm` (config 4: tcgen05 NVFP4 GEMM
8192^3 against the measured FP4 MMA peak) and `moe` (config 5: Nemotron-3-Nano
expert step per GPU, quantize + grouped GEMMs).

`--impl reference` times the reference algorithm's CPU implementation (the
oracle port in oracle/, float64, all host threads) on a bounded sample of the
same workload and prints the same metric.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
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
C3_SEED = 1234                     # rank r's slab: torch.Generator(cuda).manual_seed(C3_SEED + r)
MOE = dict(E=16, T=3072, H=2688, F=1856)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback (B200_PROFILING.md)"


def fp4_peak():
    """Dense FP4 tcgen05 peak measured by tools/mma_rate on this pool
    (profiles/fp4_mma_peak.json), else the nominal figure."""
    p = os.path.join(ROOT, "profiles", "fp4_mma_peak.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["tflops"]), f"measured: {d.get('how', 'tools/mma_rate')}"
    return FP4_DENSE_NOMINAL_TFLOPS, "nominal dense FP4 (no measured FP4 peak)"


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


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(argv, n: int) -> int:
    """`bench.py --gpus N` without a torchrun environment: run N ranks (one
    process per GPU) under torch.distributed.run on this node and forward
    rank 0's output."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.abspath(__file__)] + list(argv)
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")        # communicator size shows in the log (stderr)
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


# ---------------------------------------------------------------------------
# workloads (shared with tests/test_gpu_headline.py, which checks exactly
# these tensors against the oracle)
# ---------------------------------------------------------------------------

def c3_slab(dev, rank: int, world: int):
    """Rank `rank`'s row slab of the config-3 activation (BF16 N(0,1))."""
    import torch

    from paper_2512_02010_b200.sharded import shard_rows

    r0, r1 = shard_rows(ROWS, world, rank)
    g = torch.Generator(device=dev).manual_seed(C3_SEED + rank)
    return torch.randn(r1 - r0, COLS, generator=g, device=dev).to(torch.bfloat16)


def c4_operands(dev, n: int = 8192):
    """Config 4: A = X[M,K], B = W[N,K], BF16 N(0,1), both K-major."""
    import torch

    g = torch.Generator(device=dev).manual_seed(0)
    xa = torch.randn(n, n, generator=g, device=dev).to(torch.bfloat16)
    xb = torch.randn(n, n, generator=g, device=dev).to(torch.bfloat16)
    return xa, xb


def moe_tensors(dev, E=None, T=None, H=None, F=None):
    """Config 5, one GPU of EP=8: per expert x [T,H], h [T,F] (activations),
    dy [T,H], dh [T,F] (gradients), W1 [F,H], W2 [H,F] (weights); stacked
    over E experts, BF16 (activations N(0,1), weights N(0,0.02^2),
    gradients N(0,1e-6))."""
    import torch

    E, T, H, F = (E or MOE["E"]), (T or MOE["T"]), (H or MOE["H"]), (F or MOE["F"])
    g = torch.Generator(device=dev).manual_seed(5)

    def r(*shape, std=1.0):
        return (torch.randn(*shape, generator=g, device=dev) * std).to(torch.bfloat16)

    return {"x": r(E, T, H), "h": r(E, T, F), "dy": r(E, T, H, std=1e-3), "dh": r(E, T, F, std=1e-3),
            "W1": r(E, F, H, std=0.02), "W2": r(E, H, F, std=0.02)}


def moe_step(t, cfg, out_dtype=None):
    """One MoE expert fwd/bwd step of the 4/6 recipe (reference qlinear.py:
    107-159) for E experts: quantize every operand with 4/6 (X, H, dY, dH 1-D
    along the contraction dim; W1, W2 in 16x16 tiles giving W and W^T; the
    WGRAD operands transposed through the 16-wide RHT along tokens), each
    expert with its own tensor scale, one grouped launch per operand kind;
    then the six grouped NVFP4 GEMMs.  Returns {name: C [E, M, N]} and the
    plan {name: (A, B, M, N, K)} of GroupedQuantized operands."""
    import torch

    import paper_2512_02010_b200 as f46

    out_dtype = out_dtype or torch.bfloat16
    spec = f46.RhtSpec(seed=cfg.seed)
    q1 = lambda a: f46.quantize_grouped(a, cfg, check_finite=False)
    q2 = lambda w: f46.quantize_weights_2d_grouped(w, cfg, check_finite=False)
    qrht = lambda a: f46.quantize_wgrad_operand_grouped(a, cfg, spec, check_finite=False)
    xq, hq, dyq, dhq = q1(t["x"]), q1(t["h"]), q1(t["dy"]), q1(t["dh"])
    w1, w2 = q2(t["W1"]), q2(t["W2"])
    dyT, hT, dhT, xT = qrht(t["dy"]), qrht(t["h"]), qrht(t["dh"]), qrht(t["x"])
    T, H = t["x"].shape[1:]
    F = t["h"].shape[2]
    plan = {
        "fprop_x_w1": (xq, w1, T, F, H),
        "fprop_h_w2": (hq, w2, T, H, F),
        "dgrad_dy_w2": (dyq, w2.transposed, T, F, H),
        "dgrad_dh_w1": (dhq, w1.transposed, T, H, F),
        "wgrad_dy_h": (dyT, hT, H, F, T),
        "wgrad_dh_x": (dhT, xT, F, H, T),
    }
    outs = {}
    for name, (a, b, M, N, K) in plan.items():
        outs[name] = f46.gemm_nvfp4_grouped(*a.operands(), *b.operands(), M, N, K, out_dtype)
    return outs, plan


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
    sample = (f"{sample_rows}x{COLS} BF16 rows of the c3 workload per step (oracle port: float64 C "
              f"restatement of the reference fp4emu algorithm, {cores} OpenMP threads; the stock "
              f"single-core numpy reference takes ~73 s for the full 65536x4096 tensor, "
              f"BASELINE.md / SURVEY.md 8(d))")
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


def timed_flushed(fn, flush, stream, n, warm=1):
    """Mean device time of fn() over n runs, each after a clean L2 flush, with
    the GPU kept busy while the host enqueues (so launch latency is not timed)."""
    import torch

    for _ in range(warm):
        fn()
    ts = []
    for i in range(n):
        flush(i)
        torch.cuda._sleep(2_000_000)  # ~1 ms: covers the host enqueue of Python-level calls
        s, e = _events(2)
        s.record(stream)
        fn()
        e.record(stream)
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return sum(ts) / len(ts)


def timed_back_to_back(fn, stream, reps, warm=2):
    import torch

    for _ in range(warm):
        fn()
    s, e = _events(2)
    torch.cuda.synchronize()
    torch.cuda._sleep(1_000_000)
    s.record(stream)
    for _ in range(reps):
        fn()
    e.record(stream)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def check_parity_c3(sq, x, rank, world, amax_global):
    """The timed step's own output against the oracle (outside the timed
    region): codes, scales and alpha bit for bit, this rank's slab with the
    global alpha -- identical to the unsharded reference call on that slab's
    rows."""
    import numpy as np
    import torch

    from oracle import oracle as O
    from paper_2512_02010_b200.blockquant import tc_to_rowmajor

    t0 = time.perf_counter()
    bits = x.cpu().view(torch.int16).numpy().view(np.uint16)
    alpha = O.tensor_scale(float(amax_global), 6.0, 256.0)
    cores = max(1, len(os.sched_getaffinity(0)) // world)
    ref = O.quantize(bits, "adaptive", alpha=alpha, nthreads=cores)
    rows = x.shape[0]
    codes_ok = np.array_equal(sq.codes.cpu().numpy(), ref["codes"])
    scales_ok = np.array_equal(tc_to_rowmajor(sq.scales_tc, rows, COLS // 16).cpu().numpy(),
                               ref["scales"])
    alpha_ok = float(sq.alpha.item()) == ref["alpha"]
    return {"ok": bool(codes_ok and scales_ok and alpha_ok), "codes": bool(codes_ok),
            "scales": bool(scales_ok), "alpha": bool(alpha_ok), "rows": rows,
            "check_s": round(time.perf_counter() - t0, 2),
            "how": "the last timed step's packed codes, tcgen05 scales and alpha vs the CPU oracle "
                   "(float64 restatement pinned to reference fixtures), bit for bit"}


def run_b200(args):
    import torch
    import torch.distributed as dist

    import paper_2512_02010_b200 as f46
    from paper_2512_02010_b200 import _lib
    from paper_2512_02010_b200.blockquant import amax_device
    from paper_2512_02010_b200.sharded import ShardedQuantizer, nccl_max_allreduce

    rank, world, local = dist_env()
    if world != args.gpus:
        print(json.dumps({"error": f"WORLD_SIZE={world} but --gpus {args.gpus}"}), flush=True)
        return 2
    if not torch.cuda.is_available() or torch.cuda.device_count() <= local:
        print(json.dumps({"error": f"rank {rank} needs cuda:{local}; "
                                   f"{torch.cuda.device_count()} device(s) visible"}), flush=True)
        return 2
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        comm = {"backend": dist.get_backend(), "nranks": dist.get_world_size(),
                "nccl_version": ".".join(map(str, torch.cuda.nccl.version()))}
    L = _lib.load()
    peaks, peaks_kind = measured_peaks()

    x = c3_slab(dev, rank, world)
    rows_local = x.shape[0]
    elems_local = x.numel()
    elems_total = ROWS * COLS
    stream = torch.cuda.current_stream()
    flush_buf = L2Flush(dev)
    sq = ShardedQuantizer(rows_local, COLS, torch.bfloat16, dev, "adaptive",
                          all_reduce_max=nccl_max_allreduce())
    k2_s, k2_e = _events(args.steps), _events(args.steps)
    s_ptr = stream.cuda_stream

    def step(i=None):
        sq.amax_local(x, s_ptr)          # K1
        sq.exchange()                    # NCCL all_reduce(MAX) of 8 bytes (world > 1)
        if i is not None:
            k2_s[i].record(stream)
        sq.quantize_local(x, s_ptr)      # K2
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
        torch.cuda._sleep(2_000_000)  # ~1 ms: device busy while the host enqueues the step
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

    # roofline of K2 (fused quantize): algorithmic bytes / mean launch time, per rank
    k2 = sum(s.elapsed_time(e) for s, e in zip(k2_s, k2_e)) / args.steps
    k2_bytes = elems_local * K2_BYTES_PER_ELEM
    k2_achieved = k2_bytes / (k2 * 1e-3) / 1e9
    per_rank = torch.tensor([k2, k2_achieved, ms], dtype=torch.float64, device=dev)
    if world > 1:
        gathered = [torch.empty_like(per_rank) for _ in range(world)]
        dist.all_gather(gathered, per_rank)
    else:
        gathered = [per_rank]
    per_rank_list = [{"rank": r, "k2_ms": float(v[0]), "k2_GB/s": float(v[1]),
                      "k2_frac": float(v[1]) / peaks["hbm_gbs"], "step_ms": float(v[2])}
                     for r, v in enumerate(gathered)]
    roofline = {"bound": "hbm", "kernel": "quant_seg_kernel<bf16,adaptive> (K2)",
                "achieved": k2_achieved, "peak": peaks["hbm_gbs"], "peak_kind": peaks_kind,
                "unit": "GB/s", "frac": k2_achieved / peaks["hbm_gbs"],
                "traffic": profile_traffic("quant_seg_kernel"),
                "algorithmic_bytes_per_launch": k2_bytes,
                "bytes_per_elem": K2_BYTES_PER_ELEM, "launch_ms": k2,
                "amax_k1_plus_allreduce_ms": ms - k2, "per_rank": per_rank_list}

    parity = check_parity_c3(sq, x, rank, world, sq.amax.item()) if not args.no_parity else None
    if parity is not None and world > 1:
        ok = torch.tensor([1 if parity["ok"] else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        parity["all_ranks_ok"] = bool(ok.item())

    # end to end through the public API with pinned host buffers, N ranks
    xh = x.cpu().pin_memory()
    cfg = f46.QuantConfig(scale_mode="adaptive")
    ar = nccl_max_allreduce()

    # Two independent steps in flight on two streams, each with its own device
    # and host output buffers: step i+1's host->device copy overlaps step i's
    # device->host read (PCIe is full duplex).  Every step still copies its
    # whole input in and its whole result out inside the timed region.
    lanes = []
    for _ in range(2):
        lanes.append({"stream": torch.cuda.Stream(device=dev),
                      "codes_h": torch.empty(sq.codes.shape, dtype=torch.uint8).pin_memory(),
                      "scales_h": torch.empty(sq.scales_tc.shape, dtype=torch.uint8).pin_memory()})

    def e2e_step(ln):
        with torch.cuda.stream(ln["stream"]):
            xd = xh.to(dev, non_blocking=True)
            a = amax_device(xd)
            if ar is not None:
                ar(a)
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
           "h2d_bytes_per_step": int(xh.numel() * 2) * world,
           "d2h_bytes_per_step": int(lanes[0]["codes_h"].numel() + lanes[0]["scales_h"].numel()) * world,
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
                   "l2": ("flushed before every timed step (256 MB write + 256 MB read sweep: L2 cold "
                          "and clean); the rank's slab is " + (
                              "512 MB > L2" if world == 1 else
                              f"{rows_local * COLS * 2 >> 20} MB, so K2's re-read of the input after "
                              "K1 may partly hit L2; bytes are still counted as two reads "
                              "(algorithmic)")),
                   "bytes_per_elem": BYTES_PER_ELEM},
        "roofline": roofline, "e2e": e2e, "parity": parity, "comm": comm,
        "gpu_launches": 2 * args.steps,
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_extras:
        line["c1"] = bench_c1(args, dev, peaks)
        line["weights"] = bench_weights(args, L, dev, peaks)
        line["dequant"] = bench_dequant(args, L, dev, peaks, sq, rows_local)
        line["gemm"] = bench_gemm(args, dev, peaks)
        line["moe"] = bench_moe(args, dev)
        line["next_rows"] = bench_next_rows(args, dev, peaks)
        line["cpu_baseline"] = cpu_baseline(args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def bench_c1(args, dev, peaks):
    """Config 1: 4/6 vs standard NVFP4 (M=6) on a 4096^2 N(0,1) BF16 tensor:
    time of each (amax + quantize, L2 flushed), the adaptive overhead, each
    mode's reconstruction MSE and the fraction of blocks that pick M=4."""
    import torch

    import paper_2512_02010_b200 as f46
    from paper_2512_02010_b200 import _lib
    from paper_2512_02010_b200.sharded import ShardedQuantizer

    x = torch.randn(4096, 4096, generator=torch.Generator().manual_seed(0)).to(torch.bfloat16).to(dev)
    stream = torch.cuda.current_stream()
    flush = L2Flush(dev)
    out = {"shape": [4096, 4096], "data": "torch.randn(Generator().manual_seed(0)) -> bf16"}
    for mode in ("fixed6", "adaptive"):
        sq = ShardedQuantizer(4096, 4096, torch.bfloat16, dev, mode,
                              fp8_cap=256.0 if mode == "adaptive" else 448.0)
        ms = timed_flushed(lambda: sq(x), flush, stream, max(5, args.steps))
        sq.amax_local(x, stream.cuda_stream)
        k2 = timed_flushed(lambda: sq.quantize_local(x, stream.cuda_stream), flush, stream,
                           max(5, args.steps))
        cfg = f46.QuantConfig(scale_mode=mode)
        q = (f46.quantize_tensor_adaptive(x, cfg, want_pick4=True) if mode == "adaptive"
             else f46.quantize_tensor(x, cfg))
        mse = f46.reconstruction_mse(x, f46.dequantize_tensor(q, torch.float64))
        out[mode] = {"ms": ms, "k2_ms": k2, "GB/s": x.numel() * BYTES_PER_ELEM / ms / 1e6,
                     "mse": mse}
        if mode == "adaptive":
            out["pick4_fraction"] = float(q.pick4.double().mean())
    out["overhead_end_to_end"] = out["adaptive"]["ms"] / out["fixed6"]["ms"]
    out["overhead_k2"] = out["adaptive"]["k2_ms"] / out["fixed6"]["k2_ms"]
    out["mse_ratio_adaptive_over_fixed6"] = out["adaptive"]["mse"] / out["fixed6"]["mse"]
    out["note"] = ("paper: 4/6 adds <15% quantization overhead (PAPER.md:82); the tensor is 32 MB "
                   "(L2-sized), L2 flushed before every timed run")
    return out


def bench_dequant(args, L, dev, peaks, sq, rows):
    """K3: dequantize the c3 tensor's codes back to bf16 / f32 (L2 flushed)."""
    import torch

    from paper_2512_02010_b200 import _lib

    stream = torch.cuda.current_stream()
    flush_buf = L2Flush(dev)
    out = {}
    for od, code, ob in ((torch.bfloat16, _lib.DT_BF16, 2), (torch.float32, _lib.DT_F32, 4)):
        y = torch.empty((rows, COLS), dtype=od, device=dev)

        def run():
            _lib.check(L.f46_dequantize(sq.codes.data_ptr(), sq.scales_tc.data_ptr(), _lib.SCALES_TC,
                                        sq.alpha.data_ptr(), rows, COLS, y.data_ptr(), code, None,
                                        stream.cuda_stream), "dequantize")

        ms = timed_flushed(run, flush_buf, stream, max(5, args.steps), warm=3)
        gbs = rows * COLS * (0.5625 + ob) / (ms * 1e-3) / 1e9
        out[str(od).split(".")[-1]] = {"ms": ms, "GB/s": gbs, "frac_of_hbm": gbs / peaks["hbm_gbs"],
                                       "bytes_per_elem": 0.5625 + ob}
    return out


def bench_weights(args, L, dev, peaks):
    """Config 2: Llama-3-8B weight shapes, one GPU, end-to-end amax + 4/6 quantize."""
    import torch

    from paper_2512_02010_b200.sharded import ShardedQuantizer

    stream = torch.cuda.current_stream()
    flush_buf = L2Flush(dev)
    out = {}
    for (r, c) in [(4096, 4096), (4096, 14336), (14336, 4096)]:
        g = torch.Generator(device=dev).manual_seed(r * 7 + c)
        w = (torch.randn(r, c, generator=g, device=dev) * 0.02).to(torch.bfloat16)
        sq = ShardedQuantizer(r, c, torch.bfloat16, dev, "adaptive")
        ms = timed_flushed(lambda: sq(w), flush_buf, stream, max(5, args.steps), warm=3)
        gbs = w.numel() * BYTES_PER_ELEM / (ms * 1e-3) / 1e9
        out[f"{r}x{c}"] = {"ms": ms, "GB/s": gbs, "frac_of_hbm": gbs / peaks["hbm_gbs"],
                           "note": "amax + fused 4/6 quantize, L2 flushed, N(0,0.02^2) bf16"}
    return out


def bench_gemm(args, dev, peaks):
    """Config 4: 8192^3 tcgen05 NVFP4 GEMM of two 4/6-quantized BF16 operands."""
    import torch

    import paper_2512_02010_b200 as f46

    M = N = K = 8192
    cfg = f46.QuantConfig(scale_mode="adaptive")
    xa, xb = c4_operands(dev, M)
    aq = f46.quantize_tensor_adaptive(xa, cfg, check_finite=False)
    bq = f46.quantize_tensor_adaptive(xb, cfg, check_finite=False)
    out = {}
    flops = 2.0 * M * N * K
    stream = torch.cuda.current_stream()
    for od, name in ((torch.bfloat16, "bf16"), (torch.float32, "f32")):
        c = torch.empty((M, N), dtype=od, device=dev)
        ms = timed_back_to_back(lambda: f46.gemm_nvfp4(aq, bq, od, out=c), stream, max(5, args.steps),
                                warm=3)
        out[name] = {"ms": ms, "TFLOP/s": flops / (ms * 1e-3) / 1e12}
    tf = out["bf16"]["TFLOP/s"]
    peak, peak_kind = fp4_peak()

    # quantize(A) + quantize(B) + GEMM through the public API, inputs resident
    def full():
        qa = f46.quantize_tensor_adaptive(xa, cfg, check_finite=False)
        qb = f46.quantize_tensor_adaptive(xb, cfg, check_finite=False)
        return f46.gemm_nvfp4(qa, qb, torch.bfloat16)

    full_ms = timed_back_to_back(full, stream, 5)

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

    chain = {name: timed_back_to_back(fn, stream, 5) for name, fn in
             (("unfused_ms", unfused), ("fused_ms", fused))}
    chain["note"] = ("GEMM 8192^3 (bf16 out) + 4/6 quantize of C for the next layer; fused = amax "
                     "from the GEMM epilogue, so the quantize reads C once")
    return {
        "metric": "4/6-NVFP4 GEMM TFLOP/s", "shape": [M, N, K], "value": tf, "unit": "TFLOP/s",
        "out": out,
        "roofline": {"bound": "tensor", "kernel": "gemm_nvfp4_pair<bf16> (tcgen05 cta_group::2)",
                     "achieved": tf, "peak": peak, "peak_kind": peak_kind,
                     "unit": "TFLOP/s", "frac": tf / peak,
                     "frac_vs_nominal_9pf": tf / FP4_DENSE_NOMINAL_TFLOPS,
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

    def timed(fn):
        return timed_flushed(fn, flush, stream, max(5, args.steps))

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
    2688, FFN 1856, 3072 tokens per expert, 16 experts per GPU.  One step =
    moe_step(): 4/6 quantization of every GEMM operand (X, H, dY, dH 1-D;
    W1, W2 as 16x16 tiles giving W and W^T; the four WGRAD operands through
    the RHT along tokens) + FPROP (x W1^T, h W2^T), DGRAD (dy W2, dh W1) and
    WGRAD (dy^T h, dh^T x) as grouped NVFP4 GEMMs.  The grouped GEMMs alone
    are also timed on pre-quantized operands."""
    import torch

    import paper_2512_02010_b200 as f46

    E, T, H, F = MOE["E"], MOE["T"], MOE["H"], MOE["F"]
    cfg = f46.QuantConfig(scale_mode="adaptive")
    t = moe_tensors(dev)
    stream = torch.cuda.current_stream()
    _, plan = moe_step(t, cfg)

    res, tot_flops, gemm_ms = {}, 0.0, 0.0
    for name, (a, b, M, N, K) in plan.items():
        run = lambda: f46.gemm_nvfp4_grouped(*a.operands(), *b.operands(), M, N, K, torch.bfloat16)
        ms = timed_back_to_back(run, stream, 5, warm=3)
        fl = 2.0 * E * M * N * K
        res[name] = {"M": M, "N": N, "K": K, "experts": E, "ms": ms, "TFLOP/s": fl / (ms * 1e-3) / 1e12}
        tot_flops += fl
        gemm_ms += ms
    step_ms = timed_back_to_back(lambda: moe_step(t, cfg), stream, 3, warm=1)
    # the quantize half by operand kind, each one grouped call over the 16
    # experts (amax pass + quantize pass), L2 flushed, bytes = algorithmic
    # HBM traffic of both passes
    peaks, _ = measured_peaks()
    flush = L2Flush(dev)
    spec = f46.RhtSpec(seed=cfg.seed)
    kinds = {
        "x_1d": (lambda: f46.quantize_grouped(t["x"], cfg, check_finite=False), t["x"].numel(), 4.5625),
        "h_1d": (lambda: f46.quantize_grouped(t["h"], cfg, check_finite=False), t["h"].numel(), 4.5625),
        "w1_2d_w_and_wt": (lambda: f46.quantize_weights_2d_grouped(t["W1"], cfg, check_finite=False),
                           t["W1"].numel(), 2 * 2 + 2 * 0.5625),
        "dy_wgrad_rht_t": (lambda: f46.quantize_wgrad_operand_grouped(t["dy"], cfg, spec, check_finite=False),
                           t["dy"].numel(), 4.5625),
    }
    qk = {}
    for name, (fn, n, bpe) in kinds.items():
        ms = timed_flushed(fn, flush, stream, 10)
        qk[name] = {"ms": ms, "GB/s": n * bpe / ms / 1e6, "frac_of_hbm": n * bpe / ms / 1e6 / peaks["hbm_gbs"],
                    "bytes_per_elem": bpe}
    return {"per_gemm": res, "gemm_TFLOP/s": tot_flops / (gemm_ms * 1e-3) / 1e12, "gemm_ms": gemm_ms,
            "step_ms": step_ms, "quantize_ms": step_ms - gemm_ms,
            "step_TFLOP/s": tot_flops / (step_ms * 1e-3) / 1e12,
            "quantize_by_kind": qk,
            "note": ("per GPU of EP=8: 8 GPUs x 8192 tokens x top-6 / 128 experts = 3072 tokens/expert; "
                     "step = quantize all operands (one grouped launch pair per operand: X, H, dY, dH 1-D; "
                     "W1, W2 2-D tiles with W^T; dY, H, dH, X transposed through the RHT for WGRAD; each "
                     "expert its own tensor scale) + 6 grouped GEMMs, rounding rne (the QuantConfig default)")}


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


def run_dry(args):
    """--dry-run: exercise the launcher and the rank/collective plumbing on CPU
    (gloo), no kernels: every rank all-reduces (MAX) its rank number."""
    import torch
    import torch.distributed as dist

    rank, world, _ = dist_env()
    if world != args.gpus:
        print(json.dumps({"error": f"WORLD_SIZE={world} but --gpus {args.gpus}"}), flush=True)
        return 2
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.tensor([float(rank)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "comm_nranks": world,
                          "allreduce_max": float(t.item()), "pid": os.getpid()}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--ref-rows", type=int, default=8192)
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(sys.argv[1:], args.gpus)
    if args.dry_run:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
