"""Generate tests/golden/golden.npz from the UNMODIFIED reference library.

Run in the build container (where /root/reference exists and
`make -C oracle ref` has built oracle/_ref/libdtq_ref.so):

    python tests/golden/make_golden.py

Every output array below is produced by the reference's own public API
(dtq::quantize, dtq::make_quant_linear, dtq::qlinear_forward,
dtq::hadamard_matrix, dtq::rotate_channels, dtq::compute_scaling_mask,
dtq::apply_scaling, dtq::pack_codes) through oracle/ref_shim.cpp.  Inputs
are drawn once with numpy PCG64 and stored as fp16 so the same bytes feed
both the checker and the GPU (std::normal_distribution
is libstdc++-specific, so inputs are never regenerated per side).

The fixture pins (1) the C restatement in oracle/dtq_oracle.c on the GPU
box, where /root/reference does not exist, and (2) the GPU path directly.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def activations(rng, M, K, outliers=4):
    """SURVEY.md section 8d input recipe: N(0,1) * log-normal channel gain,
    a few x30 outlier channels, and fixed edge rows."""
    g = np.exp(rng.standard_normal(K))
    x = rng.standard_normal((M, K)) * g
    if outliers:
        x[:, rng.choice(K, outliers, replace=False)] *= 30.0
    x = x.astype(np.float16)
    if M >= 6:
        x[0] = 0.0                      # all-zero row -> degenerate s=1, z=0
        x[1] = 0.5                      # constant row -> degenerate
        x[2] = np.abs(x[2])             # all-positive row (range widened to 0)
        x[3] = -np.abs(x[3])            # all-negative row
        x[4] = np.float16(-3.0)         # constant negative row -> z = clamp(3)
        # tie-heavy row: values on the half-grid of their own scale
        k = np.arange(K) % 255
        x[5] = (k - 127).astype(np.float16)
    return x


def main():
    ref = Reference()
    rng = np.random.default_rng(1234)
    gold: dict[str, np.ndarray] = {}

    # ---- known answers from the reference unit tests -------------------
    for name, grp, bits in [("ka_grid", np.arange(16.0), 4),          # test_quant.cpp:31-37
                            ("ka_pm1", np.array([-1.0, 1.0]), 8),     # test_quant.cpp:39-45
                            ("ka_const", np.array([5.0, 5.0, 5.0]), 8)]:  # :47-56
        s, z = ref.minmax_params(grp, bits)
        gold[f"{name}_in"] = grp
        gold[f"{name}_bits"] = np.array(bits)
        gold[f"{name}_s"] = np.array(s)
        gold[f"{name}_z"] = np.array(z)

    # ---- per-token quantizer at the PixArt width ----------------------
    K = 1152
    x = activations(rng, 64, K)
    codes, s, z = ref.quantize_rows(x.astype(np.float64), 8)
    gold.update(q_x=x, q_codes=codes, q_s=s, q_z=z)
    for bits in (2, 4, 6):
        c, s_, z_ = ref.quantize_rows(x.astype(np.float64), bits)
        gold.update({f"q{bits}_codes": c, f"q{bits}_s": s_, f"q{bits}_z": z_})

    # ---- weights: make_quant_linear W8 and W4 -------------------------
    N = 96
    w = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float16)
    bias = rng.standard_normal(N) * 0.1
    gold.update(w=w, bias=bias)
    for wb in (8, 4):
        wc, sw, zw = ref.make_quant_linear(w.astype(np.float64), wb)
        y = ref.qlinear_forward(x.astype(np.float64), wc, sw, zw, wb, bias)
        y_nb = ref.qlinear_forward(x.astype(np.float64), wc, sw, zw, wb, None)
        gold.update({f"w{wb}_codes": wc, f"w{wb}_s": sw, f"w{wb}_z": zw,
                     f"w{wb}_y": y, f"w{wb}_y_nobias": y_nb})
        if wb == 4:
            gold["w4_packed"] = ref.pack_codes(wc, 4)

    # ---- static-dynamic balance: smooth scales + blockwise Hadamard ----
    x_cal = activations(rng, 32, K).astype(np.float64)
    smooth = ref.scaling_mask(np.abs(x_cal).max(0), np.abs(w.astype(np.float64)).max(0), 0.5)
    signs = ref.hadamard_signs(K, 7)
    xs, ws = ref.apply_scaling(x.astype(np.float64), w.astype(np.float64), smooth)
    xr = ref.rotate_blocks(xs, signs, 128)
    wr = ref.rotate_blocks(ws, signs, 128)
    bc, bs, bz = ref.quantize_rows(xr, 8)
    bwc, bsw, bzw = ref.make_quant_linear(wr, 8)
    by = ref.qlinear_forward(xr, bwc, bsw, bzw, 8, bias)
    # rotation only (no smoothing)
    xr_only = ref.rotate_blocks(x.astype(np.float64), signs, 128)
    rc, rs, rz = ref.quantize_rows(xr_only, 8)
    gold.update(bal_smooth=smooth, bal_signs=signs, bal_codes=bc, bal_s=bs,
                bal_z=bz, bal_wcodes=bwc, bal_ws=bsw, bal_wz=bzw, bal_y=by,
                rot_codes=rc, rot_s=rs, rot_z=rz)

    # ---- ragged shapes (tails in every dimension) ----------------------
    for i, (m, k, n) in enumerate([(5, 40, 24), (33, 200, 17), (130, 136, 264)]):
        xx = activations(rng, m, k, outliers=1)
        ww = rng.standard_normal((n, k)).astype(np.float16)
        bb = rng.standard_normal(n)
        wc, sw, zw = ref.make_quant_linear(ww.astype(np.float64), 8)
        yy = ref.qlinear_forward(xx.astype(np.float64), wc, sw, zw, 8, bb)
        xc, xs_, xz = ref.quantize_rows(xx.astype(np.float64), 8)
        gold.update({f"rag{i}_x": xx, f"rag{i}_w": ww, f"rag{i}_b": bb, f"rag{i}_wc": wc,
                     f"rag{i}_sw": sw, f"rag{i}_zw": zw, f"rag{i}_y": yy, f"rag{i}_xc": xc,
                     f"rag{i}_xs": xs_, f"rag{i}_xz": xz})

    # ---- a quantized checkpoint written by the reference (trace_io.cpp) --
    # (own RNG so the arrays above are unchanged)
    crng = np.random.default_rng(77)
    ck_layers = []
    for i, (name, n, k, b, bal) in enumerate([("blocks.0.attn.qkv", 64, 256, 8, True),
                                              ("blocks.0.mlp.fc1", 96, 256, 4, False),
                                              ("blocks.0.mlp.fc2", 48, 128, 6, False),
                                              ("blocks.0.attn.proj", 32, 128, 2, False)]):
        wk = crng.standard_normal((n, k)) / np.sqrt(k)
        mask = (np.exp(0.3 * crng.standard_normal(k))).astype(np.float32) if bal else None
        rot = ref.hadamard_signs(k, 11) if bal else None
        ck_layers.append((name, wk, b, mask, rot))
    ck_path = os.path.join(os.path.dirname(OUT), "ckpt.bin")
    ref.write_checkpoint(ck_path, ck_layers)
    for i, (name, wk, b, mask, rot) in enumerate(ck_layers):
        n, k = wk.shape
        c, sc, zc = ref.read_checkpoint_layer(ck_path, i, n, k)
        gold.update({f"ck{i}_codes": c, f"ck{i}_s": sc, f"ck{i}_z": zc})
        if mask is not None:
            # the layer's forward as the reference composes it: X / mask, the
            # full K-point rotation (balance.cpp:57-67, 94-107), then
            # qlinear_forward over the stored codes
            xk = activations(crng, 40, k)
            xs_, _ = ref.apply_scaling(xk.astype(np.float64), wk, mask.astype(np.float64))
            xr_ = ref.rotate_blocks(xs_, rot, k)
            gold.update({f"ck{i}_mask": mask, f"ck{i}_rot": rot, f"ck{i}_x": xk,
                         f"ck{i}_y": ref.qlinear_forward(xr_, c, sc, zc, b, None)})

    np.savez_compressed(OUT, **gold)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes, {len(gold)} arrays), {ck_path} "
          f"({os.path.getsize(ck_path)} bytes)")


if __name__ == "__main__":
    main()
