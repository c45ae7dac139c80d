"""Generate tests/golden/ckpt_rot.bin + golden_rot.npz from the UNMODIFIED
reference library: checkpoint layers whose weights carry a full C_in-point
Hadamard rotation wider than the fused quantizer's 256-column blocks (the
reference's `dtq quantize` rotates by hadamard_matrix(w.cols()),
dtq_main.cpp cmd_quantize), with the reference's own balanced forward:
apply_scaling + rotate_channels over all C_in columns + qlinear_forward.

Run in the build container (needs oracle/_ref/libdtq_ref.so):
    python tests/golden/make_ckpt_rot.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from make_golden import activations  # noqa: E402
from oracle.oracle import Reference  # noqa: E402


def main():
    ref = Reference()
    rng = np.random.default_rng(512)
    layers = []
    for name, n, k, b in [("blocks.3.attn.qkv", 48, 1024, 8), ("blocks.3.mlp.fc1", 40, 512, 4)]:
        wk = rng.standard_normal((n, k)) / np.sqrt(k)
        mask = np.exp(0.3 * rng.standard_normal(k)).astype(np.float32)
        rot = ref.hadamard_signs(k, 13)
        layers.append((name, wk, b, mask, rot))
    path = os.path.join(HERE, "ckpt_rot.bin")
    ref.write_checkpoint(path, layers)
    gold = {}
    for i, (name, wk, b, mask, rot) in enumerate(layers):
        n, k = wk.shape
        c, sc, zc = ref.read_checkpoint_layer(path, i, n, k)
        x = activations(rng, 24, k)
        xs_, _ = ref.apply_scaling(x.astype(np.float64), wk, mask.astype(np.float64))
        xr = ref.rotate_blocks(xs_, rot, k)
        gold.update({f"r{i}_codes": c, f"r{i}_s": sc, f"r{i}_x": x,
                     f"r{i}_y": ref.qlinear_forward(xr, c, sc, zc, b, None)})
    out = os.path.join(HERE, "golden_rot.npz")
    np.savez_compressed(out, **gold)
    print(f"wrote {path} ({os.path.getsize(path)} bytes), {out}")


if __name__ == "__main__":
    main()
