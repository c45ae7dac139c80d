"""Block linear stacks of the DiT models the reference quantizes, run through
the device path: every linear is a PlannedLinear (a MixedPrecisionPlan row,
plan.hpp:30-40, dispatched per denoising step as toydit.cpp:113-117) with
static-dynamic channel balance (smooth + 128-block Hadamard) and, where the
model has one in front of the linear, a fused prologue:

  * LN_MODULATE (LayerNorm + adaLN t2i_modulate) before qkv / fc1,
  * GELU (toydit.cpp:83) between fc1 and fc2: by default in fc1's GEMM
    epilogue (`dtq_qlinear_forward_act`, on fp32 y before the cast), so fc2's
    quantizer runs with no prologue; `gelu_in_fc1_epilogue=False` puts it in
    fc2's quantizer prologue instead (round 1).

Data flow per block: every hidden-width linear reads the block input x
(attention itself is not on the quantized-linear path; its output is stood
in for by x), cross-attention kv reads the text tokens, fc2 reads fc1's
fp16 output, and fc2's output is the next block's x -- so the final output
depends on every block's MLP chain (the equality check of the multi-GPU
path gathers it).

Weights are random-init (no checkpoints offline), drawn from a seeded device
generator so every rank of a token-row-sharded run holds identical weights
(replicated).
"""
from __future__ import annotations

from dataclasses import dataclass

import paper_2406_02540_b200 as dtq

HIDDEN = 1152

# (name, K, N, input, prologue); input "x" = block input, "txt" = text tokens,
# "fc1" = the fc1 output
PIXART_LAYERS = [
    ("attn.qkv", HIDDEN, 3 * HIDDEN, "x", "ln_mod"),
    ("attn.proj", HIDDEN, HIDDEN, "x", None),
    ("cross.q", HIDDEN, HIDDEN, "x", None),
    ("cross.kv", HIDDEN, 2 * HIDDEN, "txt", None),
    ("cross.proj", HIDDEN, HIDDEN, "x", None),
    ("mlp.fc1", HIDDEN, 4 * HIDDEN, "x", "ln_mod"),
    ("mlp.fc2", 4 * HIDDEN, HIDDEN, "fc1", "gelu"),
]
# Open-Sora STDiT: spatial and temporal self-attention, cross-attention, MLP
STDIT_LAYERS = [
    ("spatial.qkv", HIDDEN, 3 * HIDDEN, "x", "ln_mod"),
    ("spatial.proj", HIDDEN, HIDDEN, "x", None),
    ("temporal.qkv", HIDDEN, 3 * HIDDEN, "x", "ln_mod"),
    ("temporal.proj", HIDDEN, HIDDEN, "x", None),
    ("cross.q", HIDDEN, HIDDEN, "x", None),
    ("cross.kv", HIDDEN, 2 * HIDDEN, "txt", None),
    ("cross.proj", HIDDEN, HIDDEN, "x", None),
    ("mlp.fc1", HIDDEN, 4 * HIDDEN, "x", "ln_mod"),
    ("mlp.fc2", 4 * HIDDEN, HIDDEN, "fc1", "gelu"),
]


def uniform_plan(layers, blocks: int, bits: int = 8) -> dtq.MixedPrecisionPlan:
    return dtq.MixedPrecisionPlan({f"blocks.{b}.{n}": (bits,) * dtq.NUM_RANGES
                                   for b in range(blocks) for n, *_ in layers}, float(bits))


def w4a8_mp_plan(layers, blocks: int) -> dtq.MixedPrecisionPlan:
    """An illustrative W4A8 mixed-precision plan in the reference's format:
    W4 everywhere except the alignment group (cross-attention) and the
    temporal group (temporal attention) in the first timestep range, which
    stay W8 -- the shape of a metric-decoupled allocation (PAPER.md sec.
    3.4: three layer groups, four timestep ranges).  The real plan comes
    from the reference's sensitivity search (out of scope)."""
    bits = {}
    for b in range(blocks):
        for n, *_ in layers:
            sensitive = n.startswith("cross.") or n.startswith("temporal.")
            bits[f"blocks.{b}.{n}"] = (8, 4, 4, 4) if sensitive else (4, 4, 4, 4)
    nb = sum(1 for _ in bits)
    avg = sum(sum(v) for v in bits.values()) / (dtq.NUM_RANGES * nb)
    return dtq.MixedPrecisionPlan(bits, avg)


@dataclass
class StackShape:
    img_rows: int
    txt_rows: int


class LinearStack:
    """`blocks` DiT blocks of `layers`, each linear a PlannedLinear."""

    def __init__(self, layers, blocks: int, plan: dtq.MixedPrecisionPlan, device, seed: int = 7,
                 act_bits: int = 8, hblock: int = 128, eps: float = 1e-6,
                 gelu_in_fc1_epilogue: bool = True):
        import torch
        self.layers, self.blocks, self.plan, self.dev = layers, blocks, plan, device
        self.gelu_epi = gelu_in_fc1_epilogue
        g = torch.Generator(device=device).manual_seed(seed)
        signs = {}
        self.linears = []   # per block: {name: PlannedLinear}
        self.mods = []      # per block: (scale, shift) of the adaLN modulate
        for b in range(blocks):
            blk = {}
            for name, k, n, _, _ in layers:
                if k not in signs:
                    signs[k] = torch.from_numpy(dtq.hadamard_signs(k, seed)).to(device)
                w = (torch.randn((n, k), generator=g, device=device) / k ** 0.5).half()
                smooth = torch.rand(k, generator=g, device=device, dtype=torch.float64) + 0.5
                bias = torch.randn(n, generator=g, device=device, dtype=torch.float64) * 0.02
                bal = dtq.Balance(smooth, signs[k], hblock)
                blk[name] = dtq.PlannedLinear.create(w, plan, f"blocks.{b}.{name}", act_bits,
                                                     bias=bias, balance=bal)
            self.linears.append(blk)
            sc = torch.randn(HIDDEN, generator=g, device=device) * 0.1
            sh = torch.randn(HIDDEN, generator=g, device=device) * 0.1
            self.mods.append(dtq.Prologue(dtq.PROLOGUE_LN_MODULATE, sc, sh, eps))
        self.gelu = dtq.Prologue(dtq.PROLOGUE_GELU)

    def ops(self, shape: StackShape) -> float:
        rows = {"x": shape.img_rows, "fc1": shape.img_rows, "txt": shape.txt_rows}
        return self.blocks * sum(2.0 * rows[src] * k * n for _, k, n, src, _ in self.layers)

    def buffers(self, shape: StackShape):
        """Output buffers and the shared quantizer workspace for `shape`."""
        import torch
        outs = {}
        for name, k, n, src, _ in self.layers:
            if name.endswith("fc2"):  # writes the next block's x
                continue
            rows = shape.txt_rows if src == "txt" else shape.img_rows
            key = "fc1" if name.endswith("fc1") else (src, n)
            if key not in outs:
                outs[key] = torch.empty((rows, n), dtype=torch.float16, device=self.dev)
        outs["x"] = [torch.empty((shape.img_rows, HIDDEN), dtype=torch.float16, device=self.dev)
                     for _ in range(2)]
        ws_bytes = max(self.linears[b][name].workspace_bytes(shape.img_rows)
                       for b in range(self.blocks) for name, *_ in self.layers)
        outs["ws"] = torch.zeros(ws_bytes, dtype=torch.uint8, device=self.dev)  # row flags: 0
        return outs

    def forward(self, bufs, x, txt, t: int = 0, steps: int = 1):
        """One forward of the whole stack at denoising step t of `steps`;
        returns the last block's output (a buffer of `bufs`)."""
        ws = bufs["ws"]
        cur = x
        for b, blk in enumerate(self.linears):
            nxt = bufs["x"][b % 2]
            for name, k, n, src, pro in self.layers:
                layer = blk[name].select(t, steps)
                inp = txt if src == "txt" else (bufs["fc1"] if src == "fc1" else cur)
                if name.endswith("fc1"):
                    out = bufs["fc1"]
                elif name.endswith("fc2"):
                    out = nxt
                else:
                    out = bufs[(src, n)]
                act = dtq.ACT_NONE
                if self.gelu_epi and name.endswith("fc1"):
                    act = dtq.ACT_GELU  # gelu(fc1(x)) in fc1's epilogue
                if self.gelu_epi and pro == "gelu":
                    pro = None          # ... so fc2 quantizes its input as is
                p = self.mods[b] if pro == "ln_mod" else (self.gelu if pro == "gelu" else None)
                layer.forward(inp, out=out, prologue=p, workspace=ws, activation=act)
            cur = nxt
        return cur
