"""Generate the golden fixtures in tests/golden/ by running the REAL reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports fp4emu from /root/reference/pkg/src (read-only, never copied),
feeds it seeded synthetic inputs that are exactly representable in the
storage dtype (bf16 / f32 / f64), and records the reference outputs:
alpha, scale codes, FP4 codes (packed, even index in the low nibble as in
tensor_io.py:118-123), the per-block 4-vs-6 choice (adaptive.py:60-80
_dual_pass + _select) and, for small cases, the exact float64 dequantization
(blockquant.py:363-376).  The fixtures then travel with the repo to the GPU
box, where /root/reference does not exist.

Cases follow the reference's own test vectors (SURVEY.md section 8c and
Appendix B): Table-2 worked blocks at alpha = 1, tie -> 6, zero blocks,
-0.0 and tiny negatives, underflowed scales, grid tensors, a 900.0 outlier,
tail shapes (5,), (3,7), (2,3,40), and Gaussian tensors whose alpha is
inexact (amax significand not divisible by 3) as well as exact.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, os.path.join(HERE, "..", ".."))

import fp4emu  # noqa: E402
from fp4emu import adaptive as ref_adaptive  # noqa: E402
from fp4emu import blockquant as ref_bq  # noqa: E402

from oracle.oracle import bf16_bits, bf16_to_f64, pack_codes  # noqa: E402


def philox(seed):
    return np.random.Generator(np.random.Philox(seed))


def ref_run(x_f64, mode, rule="mse", alpha=None, fp8_cap=None):
    """Run the reference on a float64 view; return dict of outputs."""
    kw = {} if fp8_cap is None else {"fp8_cap": fp8_cap}
    if mode == "adaptive":
        cfg = fp4emu.QuantConfig(scale_mode="adaptive", rule=rule, **kw)
        q = fp4emu.quantize_tensor_adaptive(x_f64, cfg, alpha=alpha)
        arr = ref_bq._validated(x_f64)
        Xb, _ = ref_bq._blockify(arr, 16)
        out = ref_adaptive._dual_pass(Xb, q.alpha, cfg, 0)
        pick4 = ref_adaptive._select(out, rule).astype(np.uint8)
    else:
        cfg = fp4emu.QuantConfig(scale_mode=mode, **kw)
        q = fp4emu.quantize_tensor(x_f64, cfg, alpha=alpha)
        pick4 = np.full(q.scale_codes.shape, 1 if mode == "fixed4" else 0, np.uint8)
    cols = x_f64.shape[-1]
    rows = x_f64.size // cols
    codes = pack_codes(np.asarray(q.codes).reshape(rows, cols))
    return q, codes, pick4


CASES = []


def add(name, x_store, mode, rule="mse", alpha=None, fp8_cap=None, keep_deq=True):
    """x_store: float32 / float64 array, or uint16 bf16 bit patterns."""
    if x_store.dtype == np.uint16:
        x64 = bf16_to_f64(x_store)
    else:
        x64 = x_store.astype(np.float64)
    q, codes, pick4 = ref_run(x64, mode, rule, alpha, fp8_cap)
    rec = dict(
        x=x_store,
        mode=np.array(mode),
        rule=np.array(rule),
        alpha_override=np.array(np.nan if alpha is None else float(alpha)),
        fp8_cap=np.array(np.nan if fp8_cap is None else float(fp8_cap)),
        alpha=np.array(q.alpha),
        scales=np.asarray(q.scale_codes, np.uint8),
        codes=codes,
        pick4=pick4,
    )
    if keep_deq:
        rec["deq"] = fp4emu.dequantize_tensor(q).reshape(-1)
    CASES.append((name, rec))


def bf16(x):
    return bf16_bits(np.asarray(x, np.float32))


def main():
    A = [10.0, 20.0, 30.0, 40.0]
    B = [15.0, 30.0, 120.0, 180.0]
    # Table 2 worked blocks embedded in zero rows, alpha = 1 (test_blockquant.py:69-119)
    t2 = np.zeros((4, 32), np.float32)
    t2[0, :4] = A
    t2[1, 16:20] = B
    t2[2, :4] = B
    t2[3, 20:24] = A
    for mode in ("adaptive", "fixed6", "fixed4"):
        add(f"table2_{mode}", t2, mode, alpha=1.0)
        add(f"table2_bf16_{mode}", bf16(t2), mode, alpha=1.0)
    # tie -> 6 and all-zero block (test_adaptive.py:43-52)
    tie = np.zeros((2, 16), np.float32)
    tie[0, :4] = 6.0
    add("tie_to_6", tie, "adaptive", alpha=1.0)
    # -0.0, tiny negatives, zero blocks, mixed
    z = np.zeros((3, 48), np.float32)
    z[0, :16] = -0.0
    z[1, 16:32] = -1e-3
    z[1, 16] = 5.0
    z[2, 32:48] = np.linspace(-2, 2, 16)
    z[2, 40] = -0.0
    for mode in ("adaptive", "fixed6", "fixed4"):
        add(f"signed_zeros_{mode}", z, mode)
        add(f"signed_zeros_bf16_{mode}", bf16(z), mode)
    # underflowed scale (test_blockquant.py:191-196): 1e-30 at alpha = 448
    add("underflow_f32_fixed6", np.full((1, 16), 1e-30, np.float32), "fixed6", alpha=448.0)
    uf = np.full((2, 32), 1e-30, np.float32)
    uf[1, :16] = -2e-30
    uf[0, 16] = 0.0
    add("underflow_f32_adaptive", uf, "adaptive", alpha=448.0)
    # m=6 underflows but m=4 does not: bmax/(alpha*6) just below 2^-10
    edge = np.zeros((1, 32), np.float32)
    edge[0, :16] = np.float32(448.0 * 6 * 2.0**-10 * 0.9)
    edge[0, 16:] = np.float32(448.0 * 5.5 * 2.0**-10)
    add("underflow_edge_adaptive", edge, "adaptive", alpha=448.0)
    # grid tensors: every value on the FP4 grid times a power of two
    g = philox(7).choice([0, 0.5, 1, 1.5, 2, 3, 4, 6], size=(8, 64)) * philox(8).choice([-1, 1], size=(8, 64))
    g[:, ::16] = 6.0
    add("grid_adaptive", (g * 0.25).astype(np.float32), "adaptive")
    add("grid_bf16_adaptive", bf16(g * 0.25), "adaptive")
    # 900.0 outlier (test_acceptance.py:116)
    o = philox(11).standard_normal((16, 64)).astype(np.float32)
    o[3, 17] = 900.0
    add("outlier_bf16_adaptive", bf16(o), "adaptive")
    # max block at 4 -> scale 384 (test_adaptive.py:114-123)
    mb = philox(12).standard_normal((4, 32)).astype(np.float32)
    mb[0, :16] = np.float32(1536.0) * np.array([1, 0.75] + [0.5] * 14, np.float32)
    add("maxblock_adaptive", mb, "adaptive")
    # tail shapes (test_blockquant.py:148-153)
    for shp in [(5,), (3, 7), (2, 3, 40), (1, 16), (17, 33)]:
        xs = philox(1).standard_normal(shp).astype(np.float32)
        tag = "x".join(map(str, shp))
        add(f"tail_{tag}_adaptive", xs, "adaptive")
        add(f"tail_{tag}_bf16_fixed6", bf16(xs), "fixed6")
    # Gaussian BF16 tensors; seeds chosen to give inexact and exact alpha
    for seed in range(6):
        xg = philox(100 + seed).standard_normal((128, 256)).astype(np.float32)
        add(f"gauss_bf16_s{seed}_adaptive", bf16(xg), "adaptive", keep_deq=(seed < 2))
        if seed < 2:
            add(f"gauss_bf16_s{seed}_fixed6", bf16(xg), "fixed6", keep_deq=False)
            add(f"gauss_bf16_s{seed}_fixed4", bf16(xg), "fixed4", keep_deq=False)
    # forced amax values: inexact alpha (5.75, 5.3125, 5.1875) and exact (5.25, 5.4375, 4.875)
    for am in (5.75, 5.3125, 5.1875, 5.25, 5.4375, 4.875):
        xg = philox(int(am * 1000)).standard_normal((128, 128)).astype(np.float32)
        xg = np.clip(xg, -4.5, 4.5)
        xg[5, 7] = -am
        add(f"amax_{am}_bf16_adaptive", bf16(xg), "adaptive", keep_deq=False)
    # weight-like N(0, 0.02^2)
    w = (philox(200).standard_normal((256, 256)) * 0.02).astype(np.float32)
    add("weight_bf16_adaptive", bf16(w), "adaptive", keep_deq=False)
    # larger bf16 tensor with inexact alpha (near-tie stress)
    xl = philox(300).standard_normal((512, 1024)).astype(np.float32)
    add("gauss_bf16_512x1024_adaptive", bf16(xl), "adaptive", keep_deq=False)
    # float32 inputs
    xf = philox(400).standard_normal((128, 192)).astype(np.float32) * 3
    add("gauss_f32_adaptive", xf, "adaptive")
    add("gauss_f32_fixed6", xf, "fixed6", keep_deq=False)
    add("gauss_f32_fixed6_cap256", xf, "fixed6", fp8_cap=256.0, keep_deq=False)
    # float64 inputs as the reference's own tests use them (not f32-exact)
    x64 = philox(3).standard_normal((8, 48))
    add("gauss_f64_fixed6", x64, "fixed6")
    add("gauss_f64_adaptive", philox(5).standard_normal((16, 64)) * 2.5, "adaptive")
    add("gauss_f64_alpha_0.1", x64, "adaptive", alpha=0.1)
    # alternative selection rules (adaptive.py:77-80 with rule l1/absmax)
    for rule in ("l1", "absmax"):
        add(f"gauss_bf16_rule_{rule}", bf16(philox(500).standard_normal((64, 128))), "adaptive", rule=rule)

    out = {}
    names = []
    for name, rec in CASES:
        names.append(name)
        for k, v in rec.items():
            out[f"{name}::{k}"] = v
    out["__names__"] = np.array(names)
    path = os.path.join(HERE, "golden_quant.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {len(names)} cases to {path} ({os.path.getsize(path)/1e6:.2f} MB)")

    # 2-D 16x16 tile weight quantization (transforms.py:134-179), next row #1
    t_out = {}
    tnames = []
    for i, (shape, mode) in enumerate([((64, 96), "adaptive"), ((40, 50), "adaptive"),
                                        ((48, 32), "fixed6"), ((33, 17), "fixed4")]):
        W = bf16(philox(600 + i).standard_normal(shape) * 0.05)
        W64 = bf16_to_f64(W)
        cfg = fp4emu.QuantConfig(scale_mode=mode)
        q = fp4emu.quantize_weights_2d(W64, cfg)
        name = f"tile2d_{shape[0]}x{shape[1]}_{mode}"
        tnames.append(name)
        t_out[f"{name}::x"] = W
        t_out[f"{name}::mode"] = np.array(mode)
        t_out[f"{name}::alpha"] = np.array(q.alpha)
        t_out[f"{name}::scales"] = np.asarray(q.scale_codes, np.uint8)
        t_out[f"{name}::codes"] = pack_codes(np.asarray(q.codes))
    t_out["__names__"] = np.array(tnames)
    path = os.path.join(HERE, "golden_tile2d.npz")
    np.savez_compressed(path, **t_out)
    print(f"wrote {len(tnames)} tile cases to {path}")

    # emulated GEMM (qlinear.py:74-93) on small shapes, reference f32 k-ordered
    g_out = {}
    gnames = []
    for i, (M, N, K) in enumerate([(32, 48, 64), (64, 64, 128), (16, 40, 96)]):
        a = bf16(philox(700 + i).standard_normal((M, K)))
        b = bf16(philox(800 + i).standard_normal((N, K)))
        cfg = fp4emu.QuantConfig(scale_mode="adaptive")
        aq = fp4emu.quantize_tensor_adaptive(bf16_to_f64(a), cfg)
        bq = fp4emu.quantize_tensor_adaptive(bf16_to_f64(b), cfg)
        c = fp4emu.emulated_fp4_matmul(aq, bq, transpose_b=True)
        name = f"gemm_{M}x{N}x{K}"
        gnames.append(name)
        g_out[f"{name}::a"] = a
        g_out[f"{name}::b"] = b
        g_out[f"{name}::c"] = c
    g_out["__names__"] = np.array(gnames)
    path = os.path.join(HERE, "golden_gemm.npz")
    np.savez_compressed(path, **g_out)
    print(f"wrote {len(gnames)} gemm cases to {path}")


def linear_cases():
    """Reference linear_forward / linear_dgrad (qlinear.py:107-135) on bf16-exact inputs."""
    out, names = {}, []
    for i, (B, IN, OUT, mode) in enumerate([(32, 64, 48, "adaptive"), (48, 96, 80, "fixed6"),
                                             (40, 160, 64, "adaptive")]):
        x = bf16(philox(900 + i).standard_normal((B, IN)))
        W = bf16(philox(950 + i).standard_normal((OUT, IN)) * 0.05)
        dy = bf16(philox(980 + i).standard_normal((B, OUT)))
        cfg = fp4emu.QuantConfig(scale_mode=mode)
        y = fp4emu.linear_forward(bf16_to_f64(x), bf16_to_f64(W), cfg)
        dx = fp4emu.linear_dgrad(bf16_to_f64(dy), bf16_to_f64(W), cfg)
        name = f"linear_{B}x{IN}x{OUT}_{mode}"
        names.append(name)
        for k, v in dict(x=x, W=W, dy=dy, y=y, dx=dx, mode=np.array(mode)).items():
            out[f"{name}::{k}"] = v
    out["__names__"] = np.array(names)
    path = os.path.join(HERE, "golden_linear.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {len(names)} linear cases to {path}")


def io_and_stats_cases():
    """Reference NVF4 files (tensor_io.py:136-147) and selection_stats (adaptive.py:159-187)."""
    import tempfile

    out, names = {}, []
    cases = [((64, 128), "adaptive", 1), ((33, 20), "fixed6", 2), ((5, 7), "adaptive", 3),
             ((2, 3, 40), "fixed4", 4), ((16, 30), "adaptive", 5)]
    for shape, mode, seed in cases:
        x = bf16(philox(1000 + seed).standard_normal(shape) * 2.0)
        x64 = bf16_to_f64(x)
        if mode == "adaptive":
            cfg = fp4emu.QuantConfig(scale_mode="adaptive")
            q = fp4emu.quantize_tensor_adaptive(x64, cfg)
        else:
            q = fp4emu.quantize_tensor(x64, fp4emu.QuantConfig(scale_mode=mode))
        with tempfile.NamedTemporaryFile(suffix=".nvf") as fh:
            fp4emu.write_quantized(fh.name, q)
            raw = np.frombuffer(open(fh.name, "rb").read(), dtype=np.uint8)
        name = f"nvf4_{'x'.join(map(str, shape))}_{mode}"
        names.append(name)
        rec = dict(x=x, mode=np.array(mode), file=raw)
        if mode == "adaptive":
            st = fp4emu.selection_stats(x64, fp4emu.QuantConfig(scale_mode="adaptive"))
            rec["frac"] = np.array([st.fraction_4[r] for r in ("mse", "l1", "absmax")])
            rec["dis"] = np.array([st.disagreements[k] for k in ("mse_vs_l1", "mse_vs_absmax", "l1_vs_absmax")])
            rec["agg"] = np.array([st.aggregate_mse[r] for r in ("mse", "l1", "absmax")])
            rec["nblocks"] = np.array(st.n_blocks)
        for k, v in rec.items():
            out[f"{name}::{k}"] = v
    out["__names__"] = np.array(names)
    path = os.path.join(HERE, "golden_io.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {len(names)} io/stats cases to {path}")


def sr_rht_cases():
    """Stochastic rounding (blockquant.py:253-257), the RHT (transforms.py:92-105)
    and the gradient recipes with rounding='sr' (qlinear.py:123-159)."""
    out, names = {}, []

    def put(name, **rec):
        names.append(name)
        for k, v in rec.items():
            out[f"{name}::{k}"] = v

    for i, (shape, mode, seed, tag) in enumerate([((64, 128), "adaptive", 5, 1),
                                                   ((33, 40), "fixed6", 7, 2),
                                                   ((16, 48), "fixed4", 0, 3),
                                                   ((128, 256), "adaptive", 11, 0)]):
        x = bf16(philox(1100 + i).standard_normal(shape))
        cfg = fp4emu.QuantConfig(scale_mode=mode, rounding="sr", seed=seed)
        x64 = bf16_to_f64(x)
        if mode == "adaptive":
            q = fp4emu.quantize_tensor_adaptive(x64, cfg, sr_tag=tag)
        else:
            q = fp4emu.quantize_tensor(x64, cfg, sr_tag=tag)
        put(f"sr_{'x'.join(map(str, shape))}_{mode}_s{seed}_t{tag}", x=x, mode=np.array(mode),
            seed=np.array(seed), tag=np.array(tag), alpha=np.array(q.alpha),
            scales=np.asarray(q.scale_codes, np.uint8), codes=pack_codes(np.asarray(q.codes).reshape(shape[0], -1)))
    for i, seed in enumerate((0, 5)):
        x = philox(1200 + i).standard_normal((24, 64))
        spec = fp4emu.RhtSpec(seed=seed)
        put(f"rht_s{seed}", x=x, seed=np.array(seed), y=fp4emu.apply_rht(x, spec),
            inv=fp4emu.invert_rht(x, spec))
    for i, (B, IN, OUT, mode) in enumerate([(32, 64, 48, "adaptive"), (48, 96, 80, "fixed6")]):
        x = bf16(philox(1300 + i).standard_normal((B, IN)))
        W = bf16(philox(1350 + i).standard_normal((OUT, IN)) * 0.05)
        dy = bf16(philox(1380 + i).standard_normal((B, OUT)))
        cfg = fp4emu.QuantConfig(scale_mode=mode, rounding="sr", seed=3)
        dx = fp4emu.linear_dgrad(bf16_to_f64(dy), bf16_to_f64(W), cfg)
        dw = fp4emu.linear_wgrad(bf16_to_f64(dy), bf16_to_f64(x), cfg)
        put(f"grad_{B}x{IN}x{OUT}_{mode}", x=x, W=W, dy=dy, dx=dx, dw=dw, mode=np.array(mode))
    out["__names__"] = np.array(names)
    path = os.path.join(HERE, "golden_sr.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {len(names)} sr/rht cases to {path}")


def block_api_cases():
    """The block-level API at any length and target (blockquant.py:225-236
    compute_block_scale, :379-414 quantize_block incl. stochastic rounding
    with explicit uniforms, adaptive.py:104-146 quantize_block_adaptive per
    rule) and emulated_fp4_matmul with transpose_b=False (qlinear.py:74-93,
    the ordered float32 accumulation)."""
    out, names = {}, []

    def put(name, **rec):
        names.append(name)
        for k, v in rec.items():
            out[f"{name}::{k}"] = v

    rng = philox(1500)
    lengths = (1, 3, 7, 8, 13, 16, 17, 33, 129, 300)
    for i, n in enumerate(lengths):
        x = rng.standard_normal(n) * np.exp(rng.standard_normal() * 2)
        if i == 2:
            x[1] = -0.0
        alpha = float(np.float32(np.max(np.abs(x)) / 1536.0)) * (1.0 + 2.0 ** -20 * i)
        u = rng.random(n)
        for m in (6.0, 4.0, 5.5, 3.0):
            for rounding in ("rne", "sr"):
                r = ref_bq.quantize_block(x, alpha, m, rounding=rounding, u=u if rounding == "sr" else None)
                put(f"qb_n{n}_m{m}_{rounding}", x=x, alpha=np.array(alpha), m=np.array(m),
                    rounding=np.array(rounding), u=u, codes=np.asarray(r.codes, np.uint8),
                    scale=np.array(r.scale_code), err=np.array([r.err_mse, r.err_l1, r.err_max]),
                    deq=np.asarray(r.dequant, np.float64),
                    cbs=np.array(int(ref_bq.compute_block_scale(x, alpha, m))))
        u4 = rng.random(n)
        for rule in ("mse", "l1", "absmax"):
            for rounding in ("rne", "sr"):
                r = ref_adaptive.quantize_block_adaptive(x, alpha, rule=rule, rounding=rounding,
                                                         u6=u if rounding == "sr" else None,
                                                         u4=u4 if rounding == "sr" else None)
                put(f"qba_n{n}_{rule}_{rounding}", x=x, alpha=np.array(alpha), rule=np.array(rule),
                    rounding=np.array(rounding), u6=u, u4=u4, codes=np.asarray(r.codes, np.uint8),
                    scale=np.array(r.scale_code), m=np.array(r.chosen_m),
                    err=np.array([r.err_mse, r.err_l1, r.err_max]))
    # Table-2 blocks at alpha = 1 (test_acceptance.py:46-75)
    for name, blk in (("A", [10.0, 20.0, 30.0, 40.0]), ("B", [15.0, 30.0, 120.0, 180.0])):
        for m in (6.0, 4.0):
            r = ref_bq.quantize_block(np.array(blk), 1.0, m)
            put(f"table2_{name}_m{m}", x=np.array(blk), alpha=np.array(1.0), m=np.array(m),
                rounding=np.array("rne"), u=np.zeros(4), codes=np.asarray(r.codes, np.uint8),
                scale=np.array(r.scale_code), err=np.array([r.err_mse, r.err_l1, r.err_max]),
                deq=np.asarray(r.dequant, np.float64),
                cbs=np.array(int(ref_bq.compute_block_scale(np.array(blk), 1.0, m))))
    # transpose_b=False: A [M,K] blocked along K, B [K,N] blocked along N
    for i, (M, K, N) in enumerate([(24, 64, 40), (17, 48, 33)]):
        a = bf16_to_f64(bf16(philox(1600 + i).standard_normal((M, K))))
        b = bf16_to_f64(bf16(philox(1650 + i).standard_normal((K, N)) * 0.3))
        cfg = fp4emu.QuantConfig(scale_mode="adaptive")
        aq = fp4emu.quantize_tensor_adaptive(a, cfg)
        bq = fp4emu.quantize_tensor_adaptive(b, cfg)
        c = fp4emu.emulated_fp4_matmul(aq, bq, transpose_b=False)
        c16 = fp4emu.emulated_fp4_matmul(aq, bq, transpose_b=False, bf16_out=True)
        put(f"mm_nn_{M}x{K}x{N}", a=bf16_bits(a.astype(np.float32)), b=bf16_bits(b.astype(np.float32)),
            c=np.asarray(c, np.float32), c16=np.asarray(c16, np.float32))
    out["__names__"] = np.array(names)
    path = os.path.join(HERE, "golden_block.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {len(names)} block-api cases to {path}")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "sr":
        sr_rht_cases()
    elif len(sys.argv) > 1 and sys.argv[1] == "linear":
        linear_cases()
    elif len(sys.argv) > 1 and sys.argv[1] == "io":
        io_and_stats_cases()
    elif len(sys.argv) > 1 and sys.argv[1] == "block":
        block_api_cases()
    else:
        main()
        linear_cases()
        io_and_stats_cases()
        sr_rht_cases()
        block_api_cases()
