"""Quantized checkpoints: the reference's
read_checkpoint (trace_io.cpp:263-316) straight onto the device.

tests/golden/ckpt.bin was written by the reference's own write_checkpoint
(tests/golden/make_golden.py): W8 with a scaling mask and rotation, W4, W6
and W2 layers.  The parser is host code (CPU tests, including the
reference's FormatError cases); loading uploads the packed codes as stored
and unpacks them on the device (GPU tests, bit-exact against the
reference's read_checkpoint and forward).
"""
import os
import shutil

import numpy as np
import pytest

import paper_2406_02540_b200 as dtq

HERE = os.path.dirname(os.path.abspath(__file__))
CKPT = os.path.join(HERE, "golden", "ckpt.bin")
LAYERS = [("blocks.0.attn.qkv", 64, 256, 8, 256, 256), ("blocks.0.mlp.fc1", 96, 256, 4, 0, 0),
          ("blocks.0.mlp.fc2", 48, 128, 6, 0, 0), ("blocks.0.attn.proj", 32, 128, 2, 0, 0)]


def _lib_built():
    return os.path.exists(dtq.LIB_PATH)


pytestmark = pytest.mark.skipif(not _lib_built(), reason="libdtq_b200.so not built")


def test_checkpoint_header_and_layers():
    ck = dtq.Checkpoint(CKPT)
    assert len(ck) == len(LAYERS)
    for i, (name, n, k, bits, mlen, rlen) in enumerate(LAYERS):
        inf = ck.info(i)
        assert inf == {"name": name, "N": n, "K": k, "bits": bits, "symmetric": True,
                       "mask_len": mlen, "rot_len": rlen}
    with pytest.raises(ValueError):
        ck.info(len(LAYERS))


def _write(tmp_path, data: bytes, name="bad.bin"):
    p = tmp_path / name
    p.write_bytes(data)
    return str(p)


def test_checkpoint_format_errors(tmp_path):
    good = open(CKPT, "rb").read()
    # bad magic, bad version, truncation anywhere, trailing bytes -> FormatError
    with pytest.raises(ValueError, match="magic"):
        dtq.Checkpoint(_write(tmp_path, b"XTQCKPT\0" + good[8:]))
    bad_version = good[:8] + (2).to_bytes(2, "little") + good[10:]
    with pytest.raises(ValueError, match="version"):
        dtq.Checkpoint(_write(tmp_path, bad_version))
    for cut in (5, 12, 40, len(good) // 2, len(good) - 1):
        with pytest.raises(ValueError):
            dtq.Checkpoint(_write(tmp_path, good[:cut], f"cut{cut}.bin"))
    with pytest.raises(ValueError, match="trailing"):
        dtq.Checkpoint(_write(tmp_path, good + b"\0"))
    with pytest.raises(ValueError):
        dtq.Checkpoint(str(tmp_path / "missing.bin"))


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(len(LAYERS)))
def test_checkpoint_layers_load_bitexact(golden, i):
    ck = dtq.Checkpoint(CKPT)
    layer = ck.load(i)
    codes, scale, _ = layer.export()
    assert np.array_equal(codes, golden[f"ck{i}_codes"])
    assert np.array_equal(scale, golden[f"ck{i}_s"])


@pytest.mark.gpu
def test_checkpoint_balanced_layer_forward_bitexact(golden):
    import torch
    ck = dtq.Checkpoint(CKPT)
    layer = ck.load(0)  # mask + full 256-point rotation, as stored
    x = torch.from_numpy(golden["ck0_x"]).to(torch.float64).cuda()
    y = layer.forward(x, mode=dtq.MODE_EXACT, out_dtype=torch.float64)
    assert np.array_equal(y.cpu().numpy(), golden["ck0_y"])


CKPT_ROT = os.path.join(HERE, "golden", "ckpt_rot.bin")


@pytest.mark.gpu
@pytest.mark.parametrize("i", [0, 1])
def test_checkpoint_full_width_rotation_forward_bitexact(i):
    # tests/golden/make_ckpt_rot.py: weights rotated by the full C_in-point
    # Hadamard (1024 and 512 columns, wider than the fused quantizer's
    # blocks), as the reference's `dtq quantize` stores them.  The loaded
    # layer rotates its activations with the same full-width rotation (fp64
    # pre-pass), bit-exact against the reference's balanced forward.
    import torch
    g = dict(np.load(os.path.join(HERE, "golden", "golden_rot.npz")))
    ck = dtq.Checkpoint(CKPT_ROT)
    layer = ck.load(i)
    codes, scale, _ = layer.export()
    assert np.array_equal(codes, g[f"r{i}_codes"]) and np.array_equal(scale, g[f"r{i}_s"])
    x = torch.from_numpy(g[f"r{i}_x"]).cuda()
    for mode in (dtq.MODE_EXACT, dtq.MODE_FAST):  # wide blocks always run in fp64
        y = layer.forward(x, mode=mode, out_dtype=torch.float64)
        assert np.array_equal(y.cpu().numpy(), g[f"r{i}_y"])
    y16 = layer.forward(x, out_dtype=torch.float16).double().cpu().numpy()
    assert np.abs(y16 - g[f"r{i}_y"]).max() <= 1e-3 * np.abs(g[f"r{i}_y"]).max()


@pytest.mark.gpu
def test_checkpoint_rotation_block_must_match_storage():
    # a block-diagonal activation rotation against fully rotated weights
    # would be silently wrong: any hblock other than 0 / the stored length
    # is rejected
    ck = dtq.Checkpoint(CKPT_ROT)
    with pytest.raises(ValueError, match="rotation length"):
        ck.load(0, hblock=128)
    ck.load(0, hblock=1024).close()
