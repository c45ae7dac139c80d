"""Benchmark of the B200 quantized-linear hot path.

N = 1 (BASELINE.json configs[1], the headline): one W8A8 quantized linear at
the PixArt-alpha 1024px fc1 shape, M=4096 tokens x K=1152 -> N=4608, with
static-dynamic channel balancing (smooth scales + 128-blockwise Hadamard)
fused into the per-token activation quantizer, fp16 in / fp16 out:
    fused quantizer (fq_tile_kernel)  ->  tcgen05 i8 GEMM + dequant epilogue (qgemm_kernel)
Inputs are resident in HBM and larger than L2: the K timed steps run back to
back over a ring of layers (each with its own weights) and x / y buffers,
>300 MB in total, captured once as a CUDA graph.  Side measurements: the C4
28-block PixArt-alpha stack (W8A8 and a W4A8 mixed-precision plan, against
FP16 cuBLAS), the C3 W4A8 shapes, and C5 on one GPU.

N > 1 (torchrun; BASELINE.json configs[4]): the headline is C5 -- the
Open-Sora STDiT 28-block linear stack over 131072 token rows, rows sharded
across the ranks (shard.row_range), weights replicated, no collective in the
timed region; value = total ops / max-over-ranks step time (strong
scaling).  After timing the final outputs are NCCL-all-gathered and rank 0
compares them bitwise with its own single-GPU forward of all rows (timed:
the 1-GPU point of the same curve).

`value`  = whole-job INT8 TOPS
`e2e`    = the same metric through the public API with pinned host buffers
           (H2D + D2H inside the timed region)
`--impl reference` times the reference's own CPU implementation
(oracle/_ref/libdtq_ref.so, compiled from the reference sources) on the
host cores, on a bounded row sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

M, K, N = 4096, 1152, 4608
WBITS, ABITS, HBLOCK = 8, 8, 128
METRIC = "quant-linear INT8 TOPS + STDiT block-linear latency vs FP16 cuBLAS, 1/2/4/8 GPU"
WORKLOAD = ("W8A8 quantized linear, PixArt-alpha 1024px fc1 (M=4096, K=1152, N=4608), "
            "smooth + 128-block Hadamard fused into the per-token quantizer, fp16 in/out")


def c2_config(world: int) -> dict:
    """The headline workload's config, identical on both arms."""
    return {"workload": WORKLOAD, "M_per_rank": M, "K": K, "N": N,
            "global_batch": M * world, "seq_len": M, "parallelism": f"dp{world}",
            "weights": "W8 per-out-channel symmetric, random init",
            "l2": "inputs larger than L2: a ring of layers (own weights) and x/y buffers "
                  "over > 300 MB, steps back to back"}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


def make_inputs(seed: int = 1234, rows: int = M):
    """SURVEY.md section 8d recipe: N(0,1) x log-normal channel gains, 4 outlier
    channels x30; W ~ N(0, 1/sqrt(K)); smooth from a separate calibration draw
    (alpha 0.5); signs from std::mt19937_64(7)."""
    rng = np.random.default_rng(seed)
    g = np.exp(rng.standard_normal(K))
    out_ch = rng.choice(K, 4, replace=False)
    x = rng.standard_normal((rows, K)) * g
    x[:, out_ch] *= 30
    x = x.astype(np.float16)
    w = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float16)
    xcal = rng.standard_normal((512, K)) * g
    xcal[:, out_ch] *= 30
    a = np.abs(xcal).max(0)
    b = np.abs(w.astype(np.float64)).max(0)
    smooth = np.where((a > 0) & (b > 0), np.clip(a ** 0.5 / b ** 0.5, 1e-5, 1e5), 1.0)
    return x, w, smooth


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region.

    NVML (nvidia-ml-py) polled from a thread every ~0.1 ms plus the query
    time -- the timed region can be under a millisecond -- with
    `nvidia-smi -lms 20` as the fallback.
    """

    # nvmlClocksEventReason* bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40}
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.nv = None
        self.samples = []   # (sm_mhz, max_mhz, set(reasons))
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._poll, daemon=True)
        except Exception:
            self.nv = None
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits", "-lms", "20"],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self.t = threading.Thread(target=self._read, daemon=True)
            except Exception:
                self.proc = None
                return self
        self.t.start()
        t0 = time.time()
        while not self.samples and time.time() - t0 < 5.0:  # sampler up before timing
            time.sleep(0.001)
        self.samples.clear()
        return self

    def _poll(self):
        nv = self.nv
        get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop.is_set():
            try:
                sm = float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = int(get_r(self.h))
                self.samples.append((sm, self.mx, {n for n, b in self.BITS.items() if r & b}))
            except Exception:
                pass
            time.sleep(0.0001)

    def _read(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.proc.stdout:
            f = [t.strip() for t in ln.strip().split(",")]
            if len(f) < 9:
                continue
            try:
                sm, mx = float(f[1]), float(f[2])
            except ValueError:
                continue
            self.samples.append((sm, mx, {n for n, v in zip(names, f[5:9])
                                          if v.lower() == "active"}))

    def __exit__(self, *a):
        self.stop.set()
        if self.nv is not None:
            self.t.join(timeout=2)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        reasons = set().union(*[s[2] for s in self.samples])
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.samples[-1][1],
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml" if self.nv is not None else "nvidia-smi"}


# DTQ_BENCH_SINGLE_GPU_RANKS=1 (path check only, never a bench number):
# every rank on cuda:0 and gloo for the collectives, so the N > 1 code path
# runs end to end on a one-GPU box (the kernels of different ranks never
# wait on each other)
_SINGLE_GPU_RANKS = os.environ.get("DTQ_BENCH_SINGLE_GPU_RANKS") == "1"


def dist_setup():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if _SINGLE_GPU_RANKS:
        local = 0
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if _SINGLE_GPU_RANKS:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cpu" if _SINGLE_GPU_RANKS else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ---------------------------------------------------------------------- C5 (multi-GPU)
# BASELINE configs[4]: Open-Sora STDiT 16 frames x 512^2 -> 16384 tokens per
# sample, batch 8 -> 131072 token rows (+ 8 x 120 T5 text tokens), 28 blocks
C5_IMG, C5_TXT, C5_BLOCKS = 131072, 960, 28
C5_WORKLOAD = ("Open-Sora STDiT 16-frame 512x512 28-block linear stack (9 linears/block: spatial "
               "+ temporal qkv/proj, cross q/kv/proj, fc1, fc2), batch 8 = 131072 token rows, "
               "W8A8 through MixedPrecisionPlan dispatch, smooth + 128-block Hadamard and "
               "LN-modulate / GELU prologues fused, token rows sharded across ranks")


def c5_config(world: int) -> dict:
    return {"workload": C5_WORKLOAD, "M_total": C5_IMG, "text_rows": C5_TXT, "blocks": C5_BLOCKS,
            "hidden": 1152, "global_batch": 8, "seq_len": 16384,
            "parallelism": f"dp{world} (token-row shards, weights replicated, no collective "
                           "in the timed region)",
            "weights": "W8 per-out-channel symmetric, random init",
            "l2": "inputs larger than L2 (one forward streams ~2.5 GB per GPU)"}


# ---------------------------------------------------------------------- CPU arms
def cpu_reference_sample(rows: int, threads: int, x, w, smooth, signs):
    """One bounded sample of the workload through the reference library:
    apply_scaling + rotate_channels (128 blocks) + make_quant_linear weights
    (prepared once, outside) + qlinear_forward on `rows` token rows."""
    from oracle.oracle import Reference
    ref = Reference()
    xs = x[:rows].astype(np.float64)
    wd = w.astype(np.float64)
    t0 = time.perf_counter()
    # activation side only (the weight side is prepared once, offline)
    xb, _ = ref.apply_scaling(xs, wd[:1], smooth)
    xb = ref.rotate_blocks(xb, signs, HBLOCK)
    t_bal = time.perf_counter() - t0
    wc, sw, zw = _ref_weights_cache(ref, wd, smooth, signs)
    t1 = time.perf_counter()
    ref.qlinear_forward(xb, wc, sw, zw, WBITS, None, ABITS, threads=threads)
    t_lin = time.perf_counter() - t1
    return t_bal + t_lin


_WCACHE = {}


def _ref_weights_cache(ref, wd, smooth, signs):
    key = (id(wd), wd.shape, id(smooth))
    if key not in _WCACHE:
        _, ws = ref.apply_scaling(wd[:1], wd, smooth)
        wr = ref.rotate_blocks(ws, signs, HBLOCK)
        _WCACHE[key] = ref.make_quant_linear(wr, WBITS, ABITS)
    return _WCACHE[key]


def cpu_reference_c5_sample(rows: int, threads: int):
    """A bounded sample of the C5 workload on the reference library: the 9
    linears of one STDiT block on `rows` token rows (apply_scaling +
    rotate_channels per 128 block + qlinear_forward each; cross kv on `rows`
    text rows).  Returns (ops, seconds)."""
    from oracle.oracle import Reference
    from paper_2406_02540_b200.stack import STDIT_LAYERS
    ref = Reference()
    rng = np.random.default_rng(5)
    ops, secs = 0.0, 0.0
    for name, k, n, _, _ in STDIT_LAYERS:
        x = rng.standard_normal((rows, k))
        w = rng.standard_normal((n, k)) / np.sqrt(k)
        smooth = rng.uniform(0.5, 1.5, k)
        signs = ref.hadamard_signs(k, 7)
        wc, sw, zw = _ref_weights_cache(ref, w, smooth, signs)
        t0 = time.perf_counter()
        xb, _ = ref.apply_scaling(x, w[:1], smooth)
        xb = ref.rotate_blocks(xb, signs, HBLOCK)
        ref.qlinear_forward(xb, wc, sw, zw, WBITS, None, ABITS, threads=threads)
        secs += time.perf_counter() - t0
        ops += 2.0 * rows * n * k
    return ops, secs


def run_reference(args, world, rank):
    if rank != 0:
        return
    from oracle.oracle import Reference
    threads = os.cpu_count() or 1
    if world == 1:
        x, w, smooth = make_inputs()
        # the reference's own hadamard_matrix draws (balance.cpp:69-80); nothing
        # of this repo's package runs on the reference arm
        signs = Reference().hadamard_signs(K, 7)
        rows = args.cpu_rows
        for _ in range(args.warmup):
            cpu_reference_sample(min(rows, 64), threads, x, w, smooth, signs)
        times = [cpu_reference_sample(rows, threads, x, w, smooth, signs)
                 for _ in range(args.steps)]
        t = float(np.mean(times))
        tops = 2.0 * rows * N * K / t / 1e12
        config = c2_config(1)
        sample = (f"{rows} of {M} token rows per step (row-local, exact), apply_scaling + "
                  "rotate_channels + qlinear_forward; ms_per_step is that sample's measured time")
        scaling = "weak"
    else:
        rows = max(16, args.cpu_rows // 8)
        for _ in range(args.warmup):
            cpu_reference_c5_sample(16, threads)
        res = [cpu_reference_c5_sample(rows, threads) for _ in range(args.steps)]
        t = float(np.mean([r[1] for r in res]))
        tops = res[0][0] / t / 1e12
        config = c5_config(world)
        sample = (f"{rows} of {C5_IMG} token rows of one STDiT block's 9 linears per step "
                  "(row-local, exact), apply_scaling + rotate_channels + qlinear_forward each; "
                  "ms_per_step is that sample's measured time")
        scaling = "strong"
    out = {
        "metric": METRIC, "impl": "reference", "value": tops, "unit": "TOPS",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "int64", "data": "synthetic", "config": config,
        "cpu_baseline": {"value": tops, "unit": "TOPS", "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": tops, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------- helpers
def graph_of(fn):
    """Capture fn() once as a CUDA graph (warmed eagerly first)."""
    import torch
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    return g


def time_graph(g, reps: int, stream=None) -> list:
    import torch
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        g.replay()
        b.record(stream)
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) * 1e-3)
    return out


# ---------------------------------------------------------------------- block stack (C4)
STACK_BLOCKS, STACK_IMG, STACK_TXT = 28, 16384, 480


def run_stack(dev, reps: int = 10):
    """C4: the 28-block PixArt-alpha linear stack at batch 4, 1024 px
    (16384 image + 480 text tokens), every linear a PlannedLinear driven by a
    MixedPrecisionPlan: uniform W8A8, and a W4A8 mixed-precision plan (W8 for
    the cross-attention group in the first timestep range, W4 elsewhere),
    against FP16 cuBLAS with the same eager LayerNorm / modulate / GELU
    prologues, and against FP16 GEMMs alone (the lower bound of any fused
    FP16 prologue).  All captured in CUDA graphs; one forward = 196 linears."""
    import torch
    import torch.nn.functional as F
    from paper_2406_02540_b200.stack import (PIXART_LAYERS, LinearStack, StackShape,
                                             uniform_plan, w4a8_mp_plan)
    shape = StackShape(STACK_IMG, STACK_TXT)
    g = torch.Generator(device=dev).manual_seed(3)
    x = (torch.randn((STACK_IMG, 1152), generator=g, device=dev) * 2).half()
    txt = torch.randn((STACK_TXT, 1152), generator=g, device=dev).half()
    res = {}
    for key, plan, epi in (("w8a8", uniform_plan(PIXART_LAYERS, STACK_BLOCKS, 8), True),
                           ("w8a8_gelu_prologue", uniform_plan(PIXART_LAYERS, STACK_BLOCKS, 8),
                            False),
                           ("w4a8_mp", w4a8_mp_plan(PIXART_LAYERS, STACK_BLOCKS), True)):
        st = LinearStack(PIXART_LAYERS, STACK_BLOCKS, plan, dev, seed=7, gelu_in_fc1_epilogue=epi)
        bufs = st.buffers(shape)
        # denoising step 12 of 20: range 2 (the mixed plan's W4 cells)
        gr = graph_of(lambda: st.forward(bufs, x, txt, t=12, steps=20))
        res[key] = float(np.median(time_graph(gr, reps)))
        if key == "w4a8_mp":
            res["mp_avg_bits"] = plan.budget
            res["mp_w4_share"] = float(np.mean([plan.bits_for(n, 2) == 4 for n in plan.bits]))
        ops = st.ops(shape)
        del gr, bufs, st
    # FP16 comparators on the same structure (x feeds the hidden-width
    # linears, fc1 -> GELU -> fc2 chains, fc2's output is the next block's x)
    wts = [[(torch.randn((n, k), generator=g, device=dev) / k ** 0.5).half()
            for _, k, n, _, _ in PIXART_LAYERS] for _ in range(STACK_BLOCKS)]
    sc = torch.randn(1152, generator=g, device=dev).half() * 0.1
    sh = torch.randn(1152, generator=g, device=dev).half() * 0.1
    outs = {n: torch.empty((STACK_TXT if src == "txt" else STACK_IMG, n), dtype=torch.float16,
                           device=dev) for _, k, n, src, _ in PIXART_LAYERS}
    xb = [torch.empty_like(x) for _ in range(2)]
    h = torch.empty((STACK_IMG, 4608), dtype=torch.float16, device=dev)

    zb = torch.zeros(4608, dtype=torch.float16, device=dev)

    sc1 = (1 + sc).contiguous()

    def fp16(prologues: bool, gelu_epilogue: bool = False):
        nonlocal h
        cur = x
        for b in range(STACK_BLOCKS):
            for (name, k, n, src, pro), w in zip(PIXART_LAYERS, wts[b]):
                inp = txt if src == "txt" else (h if src == "fc1" else cur)
                if prologues and pro == "ln_mod" and gelu_epilogue:
                    # fused FP16 arm: LayerNorm + modulate as ONE layer_norm
                    # kernel (the modulate is its elementwise affine)
                    inp = F.layer_norm(inp, (k,), weight=sc1, bias=sh, eps=1e-6)
                elif prologues and pro == "ln_mod":
                    inp = F.layer_norm(inp, (k,), eps=1e-6) * (1 + sc) + sh
                elif prologues and pro == "gelu" and not gelu_epilogue:
                    inp = F.gelu(inp)
                if gelu_epilogue and name.endswith("fc1"):
                    # cuBLASLt's GELU epilogue (what FP16 can fuse)
                    h = torch._addmm_activation(zb, inp, w.t(), use_gelu=True)
                    continue
                out = h if name.endswith("fc1") else (xb[b % 2] if name.endswith("fc2")
                                                     else outs[n])
                torch.matmul(inp, w.t(), out=out)
            cur = xb[b % 2]

    for key, pro, ge in (("fp16_cublas", True, False), ("fp16_cublas_gemm_only", False, False),
                         ("fp16_fused", True, True)):
        try:
            gr = graph_of(lambda: fp16(pro, ge))
            res[key] = float(np.median(time_graph(gr, reps)))
            del gr
        except Exception:  # the fused-epilogue comparator is best effort
            res[key] = float("nan")
    ms = {k: v * 1e3 for k, v in res.items() if not k.startswith("mp_")}
    return {"workload": "PixArt-alpha 28-block linear stack, batch 4, 1024px (16384 image + 480 "
                        "text tokens), 196 linears/forward, every linear a PlannedLinear "
                        "(MixedPrecisionPlan dispatch at step 12 of 20), CUDA graphs",
            "ms": ms["w8a8"], "tops": ops / res["w8a8"] / 1e12,
            "gelu": "in fc1's GEMM epilogue (dtq_qlinear_forward_act); fc2 quantizes as is",
            "w8a8_gelu_in_fc2_prologue_ms": ms["w8a8_gelu_prologue"],
            "w4a8_mp_ms": ms["w4a8_mp"], "w4a8_mp_avg_bits": res["mp_avg_bits"],
            "w4a8_mp_w4_share_at_range2": res["mp_w4_share"],
            "fp16_cublas_ms": ms["fp16_cublas"],
            "fp16_fused_ms": ms["fp16_fused"],
            "fp16_cublas_gemm_only_ms": ms["fp16_cublas_gemm_only"],
            "speedup_vs_fp16_fused": res["fp16_fused"] / res["w8a8"],
            "speedup_vs_fp16": res["fp16_cublas"] / res["w8a8"],
            "speedup_vs_fp16_gemm_only": res["fp16_cublas_gemm_only"] / res["w8a8"],
            "note": "fp16_cublas: eager LN / modulate / GELU + torch.matmul; fp16_fused: "
                    "LayerNorm + modulate in one layer_norm kernel (elementwise affine = "
                    "1 + scale, shift) and fc1's GELU in cuBLASLt's epilogue; gemm_only: the "
                    "GEMMs alone, the lower bound of any fused FP16 prologue",
            "ops": ops}


# ---------------------------------------------------------------------- W4A8 (C3)
def run_w4_c3(dev, KB):
    """BASELINE configs[2]: W4A8 at the STDiT block shapes, M=4096: the GEMM
    alone on pre-quantized codes (the in-GEMM nibble unpack), and the whole
    layer (fused quantizer with smooth + 128-block Hadamard that also expands
    the weights to s8 in the workspace, then the W8A8 GEMM) beside the same
    layer at W8A8 -- CUDA-graph batches over a >L2 ring of inputs."""
    import torch
    import paper_2406_02540_b200 as dtq
    out = {}
    g = torch.Generator(device=dev).manual_seed(0)
    for name, k, n in (("qkv", 1152, 3456), ("proj", 1152, 1152), ("fc1", 1152, 4608),
                       ("fc2", 4608, 1152)):
        w = (torch.randn(n, k, generator=g, device=dev) / k ** 0.5).half()
        signs = torch.from_numpy(dtq.hadamard_signs(k, 7)).to(dev)
        smooth = torch.rand(k, generator=g, device=dev, dtype=torch.float64) + 0.5
        layer = dtq.QuantLinear.create(w, 4, 8, balance=dtq.Balance(smooth, signs, 128))
        layer8 = dtq.QuantLinear.create(w, 8, 8, balance=dtq.Balance(smooth, signs, 128))
        x = torch.randn(M, k, generator=g, device=dev).half()
        codes, s_x, z_x = layer.quantize(x)
        y = torch.empty(M, n, dtype=torch.float16, device=dev)
        nb = max(2, int(256e6 // (M * k)) + 1)
        ring = [codes.clone() for _ in range(nb)]
        xr = [x.clone() for _ in range(max(2, int(256e6 // (2 * M * k)) + 1))]
        ws = layer.workspace(M, dev)

        def gemms():
            for i in range(KB):
                layer.gemm(ring[i % nb], s_x, z_x, out=y)

        def fwds(lay=layer):
            for i in range(KB):
                lay.forward(xr[i % len(xr)], out=y, workspace=ws)

        t = float(np.median(time_graph(graph_of(gemms), 5))) / KB
        tl = float(np.median(time_graph(graph_of(fwds), 5))) / KB
        t8 = float(np.median(time_graph(graph_of(lambda: fwds(layer8)), 5))) / KB
        ops = 2.0 * M * n * k
        out[name] = {"M": M, "K": k, "N": n, "gemm_ms": t * 1e3, "gemm_tops": ops / t / 1e12,
                     "layer_ms": tl * 1e3, "layer_tops": ops / tl / 1e12,
                     "w8a8_layer_ms": t8 * 1e3, "w4_over_w8": t8 / tl}
        del ring, xr, layer8
    out["note"] = ("gemm: the standalone W4A8 GEMM on pre-quantized codes, nibbles unpacked "
                   "to s8 in smem by converter warps; layer: forward = tile quantizer that "
                   "also expands the weights to s8 in the workspace, then the W8A8 GEMM; "
                   "w4_over_w8: W4A8 / W8A8 layer throughput; fp16 out")
    return out


# ---------------------------------------------------------------------- C5
def run_c5(args, dev, world, rank, stream, local, verify=True):
    """C5: the STDiT 28-block linear stack over 131072 token rows, rows
    sharded across ranks (shard.row_range), weights replicated.  Each rank
    times its shard's forward (CUDA graph, K steps back to back); the job
    time is the max over ranks.  After timing, the final fp16 outputs are
    all-gathered over NCCL and rank 0 checks them bitwise against its own
    single-GPU forward of all 131072 rows (which it also times: the 1-GPU
    strong-scaling point, measured on the same box in the same run)."""
    import torch
    from paper_2406_02540_b200.shard import gather_rows, row_range
    from paper_2406_02540_b200.stack import STDIT_LAYERS, LinearStack, StackShape, uniform_plan
    plan = uniform_plan(STDIT_LAYERS, C5_BLOCKS, 8)
    st = LinearStack(STDIT_LAYERS, C5_BLOCKS, plan, dev, seed=11)
    g = torch.Generator(device=dev).manual_seed(2025)   # same global input on every rank
    x_all = (torch.randn((C5_IMG, 1152), generator=g, device=dev) * 2).half()
    t_all = torch.randn((C5_TXT, 1152), generator=g, device=dev).half()
    lo, hi = row_range(C5_IMG, rank, world)
    tlo, thi = row_range(C5_TXT, rank, world)
    xs, ts = x_all[lo:hi], t_all[tlo:thi]
    shape = StackShape(hi - lo, thi - tlo)
    bufs = st.buffers(shape)
    res = {}
    gr = graph_of(lambda: st.forward(bufs, xs, ts, t=12, steps=20))
    for _ in range(max(1, args.warmup - 1)):
        gr.replay()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    c5_steps = max(3, min(args.steps, 20))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(c5_steps):
            gr.replay()
        e1.record(stream)
        torch.cuda.synchronize()
    res["clocks"] = clk.summary()
    barrier(world)
    t_rank = e0.elapsed_time(e1) * 1e-3 / c5_steps
    t_job = max_over_ranks(t_rank, world)
    ops = st.ops(StackShape(C5_IMG, C5_TXT))
    res.update(steps=c5_steps, ms_per_step=t_job * 1e3, tops=ops / t_job / 1e12, ops=ops,
               rows_per_rank=hi - lo)
    y_local = st.forward(bufs, xs, ts, t=12, steps=20).clone()
    # e2e: the shard from pinned host memory, the stack, the result back
    xh = xs.cpu().pin_memory()
    th = ts.cpu().pin_memory()
    yh = torch.empty_like(y_local, device="cpu").pin_memory()
    xd = torch.empty_like(xs)
    tdv = torch.empty_like(ts)

    def e2e_step():
        xd.copy_(xh, non_blocking=True)
        tdv.copy_(th, non_blocking=True)
        yh.copy_(st.forward(bufs, xd, tdv, t=12, steps=20), non_blocking=True)

    e2e_step()
    torch.cuda.synchronize()
    barrier(world)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(c5_steps):
        e2e_step()
    b.record(stream)
    torch.cuda.synchronize()
    t_e2e = max_over_ranks(a.elapsed_time(b) * 1e-3 / c5_steps, world)
    res["e2e"] = {"value": ops / t_e2e / 1e12, "unit": "TOPS",
                  "h2d_bytes_per_step": (xs.numel() + ts.numel()) * 2,
                  "d2h_bytes_per_step": y_local.numel() * 2, "ms": t_e2e * 1e3,
                  "api": "QuantLinear.forward over the stack, pinned host in/out"}
    del gr
    if verify and world > 1:
        y_all = gather_rows(y_local.cpu() if _SINGLE_GPU_RANKS else y_local,
                            C5_IMG)   # NCCL all_gather over NVLink
        y_all = y_all.to(dev)
        ok = None
        if rank == 0:
            del bufs
            torch.cuda.empty_cache()
            fb = st.buffers(StackShape(C5_IMG, C5_TXT))
            g1 = graph_of(lambda: st.forward(fb, x_all, t_all, t=12, steps=20))
            t1 = float(np.median(time_graph(g1, 3, stream)))
            y_one = st.forward(fb, x_all, t_all, t=12, steps=20)
            ok = bool(torch.equal(y_all, y_one))
            res["one_gpu"] = {"ms_per_step": t1 * 1e3, "tops": ops / t1 / 1e12,
                              "note": "rank 0 alone over all 131072 rows, same weights/inputs"}
            res["verify"] = {"ranks": world, "outputs_identical": ok,
                             "compared": "all 131072 x 1152 fp16 final outputs (bitwise)",
                             "collective": "nccl all_gather (after timing)", "timed": False}
            del g1, fb
        barrier(world)
    del st
    torch.cuda.empty_cache()
    return res


# ---------------------------------------------------------------------- C2 (headline, N=1)
def run_c2(args, dev, world, stream, local):
    """The C2 step and its per-kernel rooflines (see the module docstring)."""
    import torch
    import paper_2406_02540_b200 as dtq
    x_np, w_np, smooth_np = make_inputs(seed=1234)
    signs = dtq.hadamard_signs(K, 7)
    x = torch.from_numpy(x_np).to(dev)
    w = torch.from_numpy(w_np).to(dev)
    bal = dtq.Balance(torch.from_numpy(smooth_np).to(dev), torch.from_numpy(signs).to(dev), HBLOCK)
    layer = dtq.QuantLinear.create(w, WBITS, ABITS, balance=bal)
    y = torch.empty((M, N), dtype=torch.float16, device=dev)
    ws = layer.workspace(M, dev)
    ldc = (K + 15) // 16 * 16
    codes = torch.empty((M, ldc), dtype=torch.uint8, device=dev)[:, :K]
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    s_x = torch.empty(M, dtype=torch.float64, device=dev)
    z_x = torch.empty(M, dtype=torch.int32, device=dev)
    for _ in range(args.warmup):
        flush.fill_(1)
        layer.quantize(x, mode=dtq.MODE_FAST, out=(codes, s_x, z_x))
        layer.gemm(codes, s_x, z_x, out=y)
        layer.forward(x, out=y, workspace=ws)
    torch.cuda.synchronize()
    r = {}

    # timed step: one layer.forward (fused quantizer -> GEMM, the GEMM launched
    # with programmatic dependent launch).  Steps run back to back over a ring
    # of layers (own weights) and input/output buffers larger than L2, so
    # every step streams its activations and weights from HBM and evicts the
    # previous step's output, as consecutive layers of a network do.
    nstep_ring = max(2, int(300e6 // (M * K * 2 + N * K + M * N * 2)) + 1)
    lring = [layer] + [dtq.QuantLinear.create(w, WBITS, ABITS, balance=bal)
                       for _ in range(nstep_ring - 1)]
    sxring = [x] + [x.clone() for _ in range(nstep_ring - 1)]
    syring = [y] + [torch.empty_like(y) for _ in range(nstep_ring - 1)]

    def k_steps():
        for i in range(args.steps):
            j = i % nstep_ring
            lring[j].forward(sxring[j], out=syring[j], workspace=ws)

    k_steps()
    torch.cuda.synchronize()
    # host cost of the API call, eager (reported; not in the timed region):
    # through the Python wrapper, and through the C ABI alone (ctypes with
    # prebuilt arguments: the cost a C/C++ caller of dtq_qlinear_forward sees,
    # plus ~1-2 us of ctypes)
    h_start = time.perf_counter()
    k_steps()
    r["h_issue"] = (time.perf_counter() - h_start) / args.steps
    torch.cuda.synchronize()
    import ctypes as C
    lib = dtq.lib()
    cargs = [(C.c_void_p(sxring[j].data_ptr()), dtq.F16, M, K, lring[j]._h, dtq.MODE_FAST, None,
              C.c_void_p(syring[j].data_ptr()), dtq.F16, N, C.c_void_p(ws.data_ptr()),
              C.c_size_t(ws.numel()), None, C.c_void_p(stream.cuda_stream))
             for j in range(nstep_ring)]
    fwd = lib.dtq_qlinear_forward
    h_start = time.perf_counter()
    for i in range(args.steps):
        fwd(*cargs[i % nstep_ring])
    r["h_issue_cabi"] = (time.perf_counter() - h_start) / args.steps
    torch.cuda.synchronize()
    # the K timed steps are captured once as a CUDA graph (the quantizer ->
    # GEMM pairs keep their programmatic-dependent-launch edges)
    g_steps = graph_of(k_steps)
    for _ in range(3):  # untimed replays: clocks and L2 in their steady state
        g_steps.replay()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t0.record(stream)
        g_steps.replay()
        t1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    r["clocks"] = clk.summary()
    r["t_fwd"] = t0.elapsed_time(t1) * 1e-3 / args.steps
    del g_steps

    # the same step with a 512 MB L2 flush before each forward
    fev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        fev[i][0].record(stream)
        layer.forward(x, out=y, workspace=ws)
        fev[i][1].record(stream)
    torch.cuda.synchronize()
    r["t_flushed"] = float(np.mean([a.elapsed_time(b) for a, b in fev])) * 1e-3
    del lring[1:], sxring[1:], syring[1:]

    # per-kernel launch durations for the roofline figures: CUDA-graph batches
    # of KB back-to-back launches over a ring of inputs larger than L2
    KB = 10
    nring = max(2, int(256e6 // (2 * M * K)) + 1)
    xring = [x.clone() for _ in range(nring)]
    cring = [torch.empty((M, ldc), dtype=torch.uint8, device=dev)[:, :K] for _ in range(nring)]
    for i in range(nring):
        layer.quantize(xring[i], mode=dtq.MODE_FAST, out=(cring[i], s_x, z_x))
    torch.cuda.synchronize()

    def fq_batch():
        for i in range(KB):
            layer.quantize(xring[i % nring], mode=dtq.MODE_FAST, out=(codes, s_x, z_x))

    def gm_batch():
        for i in range(KB):
            layer.gemm(cring[i % nring], s_x, z_x, out=y)

    reps = max(3, args.steps // KB)
    r["t_fq"] = float(np.median(time_graph(graph_of(fq_batch), reps, stream))) / KB
    r["t_gm"] = float(np.median(time_graph(graph_of(gm_batch), reps, stream))) / KB
    del xring, cring

    # the same quantizer at the stack's row count (context)
    M2 = 16384
    x16 = torch.from_numpy(make_inputs(seed=99, rows=M2)[0]).to(dev)
    nr16 = max(2, int(256e6 // (2 * M2 * K)) + 1)
    r16 = [x16.clone() for _ in range(nr16)]
    c16 = torch.empty((M2, ldc), dtype=torch.uint8, device=dev)[:, :K]
    s16 = torch.empty(M2, dtype=torch.float64, device=dev)
    z16 = torch.empty(M2, dtype=torch.int32, device=dev)

    def fq16_batch():
        for i in range(KB):
            layer.quantize(r16[i % nr16], mode=dtq.MODE_FAST, out=(c16, s16, z16))

    r["t_fq16"] = float(np.median(time_graph(graph_of(fq16_batch), 5, stream))) / KB
    del r16, x16

    # e2e: host fp16 in, host fp16 out through the C-ABI host entry point
    xh = torch.from_numpy(x_np).pin_memory()
    yh = torch.empty((M, N), dtype=torch.float16).pin_memory()
    for _ in range(max(1, args.warmup)):
        layer.forward_host(xh, yh)
    barrier(world)
    eev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    for i in range(args.steps):
        eev[i][0].record(stream)
        layer.forward_host(xh, yh)
        eev[i][1].record(stream)
    torch.cuda.synchronize()
    r["t_e2e"] = max_over_ranks(float(np.mean([a.elapsed_time(b) for a, b in eev])) * 1e-3, world)

    # FP16 cuBLAS comparator on the same shape (library call, reported only),
    # timed like our step: K back to back over a >L2 ring, one CUDA graph
    hring = [(x.clone(), w.clone(), torch.empty_like(y)) for _ in range(nstep_ring)]

    def f16_steps():
        for i in range(args.steps):
            xr, wr, yr = hring[i % nstep_ring]
            torch.matmul(xr, wr.t(), out=yr)

    r["t_f16"] = float(np.median(time_graph(graph_of(f16_steps), 3, stream))) / args.steps
    hev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        hev[i][0].record(stream)
        torch.matmul(x, w.t(), out=y)
        hev[i][1].record(stream)
    torch.cuda.synchronize()
    r["t_f16_flushed"] = float(np.mean([a.elapsed_time(b) for a, b in hev])) * 1e-3
    del hring

    # cuBLASLt int8 (torch._int_mm) on the same shape: library INT8 reference point
    r["t_i8"] = None
    try:
        a8 = torch.randint(-127, 127, (M, K), dtype=torch.int8, device=dev)
        b8 = torch.randint(-127, 127, (K, N), dtype=torch.int8, device=dev).t().contiguous().t()
        r["t_i8"] = float(np.median(time_graph(graph_of(
            lambda: [torch._int_mm(a8, b8) for _ in range(KB)]), 5, stream))) / KB
    except Exception:
        pass
    r["x_np"], r["w_np"], r["smooth_np"], r["signs"] = x_np, w_np, smooth_np, signs
    return r


def rooflines(r):
    hbm, bf16, peak_src = load_peaks()
    int8_peak = 2.0 * bf16   # dense int8 = 2x dense bf16 on B200 (4.5 vs 2.25 PF nominal)
    ops = 2.0 * M * N * K
    gemm_tops = ops / r["t_gm"] / 1e12
    fq_bytes = 2 * M * K + M * K + 12 * M
    fq_bytes16 = 2 * 16384 * K + 16384 * K + 12 * 16384
    gemm_bytes = M * K + N * K * WBITS // 8 + 2 * M * N + 12 * M + 12 * N
    traffic, ceiling = None, None
    prof = os.path.join(ROOT, "profiles", "latest_traffic.json")
    if os.path.exists(prof):
        try:
            tj = json.load(open(prof))
            traffic = tj.get("qgemm_kernel_dram_bytes")
            ceiling = tj.get("int8_ceiling_tops")
        except Exception:
            pass
    # peak: the dense INT8 tensor ceiling measured on this pool's B200s
    # (tools/int8_ceiling.cu: the GEMM's own tcgen05.mma.kind::i8 back to back
    # from smem), else 2 x the driver-measured dense bf16
    peak = float(ceiling) if ceiling else int8_peak
    roof = {"bound": "tensor", "achieved": gemm_tops, "peak": peak, "unit": "TFLOP/s",
            "frac": gemm_tops / peak, "traffic": traffic,
            "kernel": "qgemm_kernel (tcgen05.mma kind::i8)",
            "peak_source": ("measured dense INT8 ceiling (profiles/r02_int8_ceiling.json)"
                            if ceiling else f"2 x {peak_src} dense bf16 ({bf16:.1f} TF/s)"),
            "frac_of_2x_measured_bf16": gemm_tops / int8_peak,
            "frac_of_nominal_4500": gemm_tops / 4500.0, "algorithmic_bytes": gemm_bytes}
    fq = {"bound": "hbm", "achieved": fq_bytes / r["t_fq"] / 1e9, "peak": hbm, "unit": "GB/s",
          "frac": fq_bytes / r["t_fq"] / 1e9 / hbm, "ms": r["t_fq"] * 1e3, "bytes": fq_bytes,
          "peak_source": peak_src,
          "at_M16384": {"ms": r["t_fq16"] * 1e3, "achieved": fq_bytes16 / r["t_fq16"] / 1e9,
                        "frac": fq_bytes16 / r["t_fq16"] / 1e9 / hbm, "bytes": fq_bytes16,
                        "note": "same kernel at the stack's 16384 rows"}}
    # the whole step against its two floors: all its HBM bytes at the measured
    # copy bandwidth (the GEMM's output written back included, which a single
    # launch hides in L2) and its INT8 ops at the measured tensor ceiling
    step_bytes = fq_bytes + gemm_bytes - M * K      # the codes stay in L2 between the two
    floors = {"hbm_us": step_bytes / (hbm * 1e9) * 1e6, "tensor_us": ops / (peak * 1e12) * 1e6}
    step = {"bytes": step_bytes, "ops": ops, **floors,
            "step_us": r["t_fwd"] * 1e6, "step_l2_flushed_us": r["t_flushed"] * 1e6,
            "frac_of_max_floor": max(floors.values()) / (r["t_fwd"] * 1e6),
            "frac_of_sum_of_floors": sum(floors.values()) / (r["t_fwd"] * 1e6),
            "note": "max floor = perfect overlap of the memory and tensor work; sum = the "
                    "two run back to back (quantizer, then GEMM)"}
    roof["step"] = step
    return roof, fq


def cpu_baseline_c2(args, r):
    threads = os.cpu_count() or 1
    rows = args.cpu_rows
    tc = cpu_reference_sample(rows, threads, r["x_np"], r["w_np"], r["smooth_np"], r["signs"])
    return {"value": 2.0 * rows * N * K / tc / 1e12, "unit": "TOPS", "cores": threads,
            "kind": "reference",
            "sample": f"{rows} of {M} token rows (row-local, exact): reference apply_scaling "
                      "+ rotate_channels per 128 block + qlinear_forward, row-sliced threads"}


def run_ours(args, world, rank, local):
    import torch
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    ops = 2.0 * M * N * K
    r = run_c2(args, dev, world, stream, local)
    roof, fq = rooflines(r)
    kernel_ms = {"fused_quantizer": r["t_fq"] * 1e3, "qgemm": r["t_gm"] * 1e3,
                 "fused_forward_call": r["t_fwd"] * 1e3,
                 "fused_forward_call_l2_flushed": r["t_flushed"] * 1e3,
                 "host_issue_per_step": r["h_issue"] * 1e3,
                 "host_issue_per_step_c_abi": r["h_issue_cabi"] * 1e3,
                 "note": "fused_forward_call: one layer.forward per step (both kernels), K steps "
                         "back to back over a >L2 ring, captured as one CUDA graph, one event "
                         "pair; host_issue_per_step: the eager Python API call (_c_abi: the C ABI call alone, ctypes with prebuilt arguments); _l2_flushed: 512 MB "
                         "write before each step, one event pair per step; per-kernel: median "
                         "of CUDA-graph batches of back-to-back launches over a >L2 input ring"}
    c2_extra = {
        "fp16_cublas": {"ms": r["t_f16"] * 1e3, "tflops": ops / r["t_f16"] / 1e12,
                        "speedup_of_ours": r["t_f16"] / r["t_fwd"],
                        "ms_l2_flushed": r["t_f16_flushed"] * 1e3,
                        "speedup_of_ours_l2_flushed": r["t_f16_flushed"] / r["t_flushed"]},
        "int8_cublaslt": None if r["t_i8"] is None else
        {"ms": r["t_i8"] * 1e3, "tops": ops / r["t_i8"] / 1e12,
         "note": "torch._int_mm s8xs8, no epilogue"},
    }
    cpu = None
    if rank == 0 and not args.no_cpu:
        if world == 1:
            cpu = cpu_baseline_c2(args, r)
        else:
            threads = os.cpu_count() or 1
            rows = max(16, args.cpu_rows // 8)
            ops_s, secs = cpu_reference_c5_sample(rows, threads)
            cpu = {"value": ops_s / secs / 1e12, "unit": "TOPS", "cores": threads,
                   "kind": "reference",
                   "sample": f"{rows} of {C5_IMG} token rows of one STDiT block's 9 linears "
                             "(row-local, exact): reference apply_scaling + rotate_channels per "
                             "128 block + qlinear_forward, row-sliced threads"}
    if world == 1:
        t_step = r["t_fwd"]
        stack = w4 = c5 = None
        if not args.no_stack:
            try:
                stack = run_stack(dev)
            except Exception as e:  # reported, never silently replaced
                stack = {"error": repr(e)[:300]}
            try:
                w4 = run_w4_c3(dev, 10)
            except Exception as e:
                w4 = {"error": repr(e)[:300]}
            try:
                c5 = run_c5(args, dev, 1, 0, stream, local, verify=False)
            except Exception as e:
                c5 = {"error": repr(e)[:300]}
        out = {
            "metric": METRIC, "value": ops / t_step / 1e12, "unit": "TOPS", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u8xs8->s32 (fp16 in/out)", "data": "synthetic", "config": c2_config(1),
            "roofline": roof, "fused_quantizer": fq, "kernel_ms": kernel_ms, **c2_extra,
            "e2e": {"value": ops / r["t_e2e"] / 1e12, "unit": "TOPS",
                    "h2d_bytes_per_step": 2 * M * K, "d2h_bytes_per_step": 2 * M * N,
                    "ms": r["t_e2e"] * 1e3, "api": "dtq_qlinear_forward_host"},
            "stack": stack, "w4a8_c3": w4, "c5_one_gpu": c5,
            "gpu_launches": 2 * args.steps,   # fused quantizer + GEMM per timed step
            "clocks": r["clocks"], "cpu_baseline": cpu,
        }
        print(json.dumps(out), flush=True)
        return
    # N > 1: the headline is C5, token rows sharded across the ranks
    c5 = run_c5(args, dev, world, rank, stream, local, verify=True)
    if rank != 0:
        return
    layers_per_step = C5_BLOCKS * 9
    out = {
        "metric": METRIC, "value": c5["tops"], "unit": "TOPS", "n_gpus": world,
        "steps": c5["steps"], "warmup": args.warmup, "ms_per_step": c5["ms_per_step"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u8xs8->s32 (fp16 in/out)", "data": "synthetic", "config": c5_config(world),
        "roofline": roof, "fused_quantizer": fq, "kernel_ms": kernel_ms, **c2_extra,
        "roofline_note": "roofline / fused_quantizer / kernel_ms: the C2-shape kernels timed on "
                         "rank 0 in this run (the C5 stack runs the same two kernels)",
        "e2e": c5["e2e"],
        "c5": {k: v for k, v in c5.items() if k not in ("e2e", "verify", "clocks")},
        "multi_gpu_verify": c5.get("verify"),
        "gpu_launches": 2 * layers_per_step * c5["steps"],
        "clocks": c5["clocks"], "cpu_baseline": cpu,
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-rows", type=int, default=512)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-stack", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    world, rank, local = dist_setup()
    run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
