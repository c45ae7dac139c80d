"""Row flags: the forward's quantizer and GEMM run concurrently, the GEMM
consuming 128-row blocks as the quantizer publishes them (GemmArgs::ready).
The result must be bit-identical to the two stages run one after the other
(layer.quantize, then layer.gemm, which waits for the whole quantizer grid),
for ragged row counts, every fp epilogue dtype, the fused prologues, repeated
forwards on one workspace (the counters reset themselves), forwards of
different M sharing a workspace, and CUDA-graph replays."""
import os

import numpy as np
import pytest

# the row-flag path is opt-in (measured slower than the two stages back to
# back, see capi.cu row_flags_wanted); this module switches it on for its own
# process before the library reads the switch
if os.environ.get("DTQ_ROW_FLAGS") != "1":
    pytest.skip("run in its own process with DTQ_ROW_FLAGS=1 "
                "(tests/test_gpu_parity.py::test_row_flag_path_subprocess)",
                allow_module_level=True)

torch = pytest.importorskip("torch")
import paper_2406_02540_b200 as dtq  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _layer(K, N, seed, wbits=8):
    g = torch.Generator(device=DEV).manual_seed(seed)
    w = (torch.randn((N, K), generator=g, device=DEV) / K ** 0.5).half()
    signs = torch.from_numpy(dtq.hadamard_signs(K, 7)).to(DEV)
    smooth = torch.rand(K, generator=g, device=DEV, dtype=torch.float64) + 0.5
    bias = torch.randn(N, generator=g, device=DEV, dtype=torch.float64) * 0.1
    return dtq.QuantLinear.create(w, wbits, 8, bias=bias, balance=dtq.Balance(smooth, signs, 128))


def _two_stage(layer, x, dt, pro=None):
    codes, s, z = layer.quantize(x, prologue=pro)
    return layer.gemm(codes, s, z, out_dtype=dt)


@pytest.mark.parametrize("M", [1, 100, 128, 129, 1000, 4096, 16384 + 37])
@pytest.mark.parametrize("N", [1152, 4608])
def test_forward_equals_two_stage(M, N):
    K = 1152
    layer = _layer(K, N, M + N)
    x = (torch.randn((M, K), device=DEV) * 3).half()
    ws = layer.workspace(M, DEV)
    for dt in (torch.float16, torch.bfloat16, torch.float32):
        want = _two_stage(layer, x, dt)
        for _ in range(3):  # the counters must be back at zero after each forward
            y = layer.forward(x, out_dtype=dt, workspace=ws)
            assert torch.equal(y, want), (M, N, dt)
    assert int(ws[:8192 * 4 + 4].count_nonzero()) == 0


@pytest.mark.parametrize("pro", ["mod", "ln", "gelu"])
def test_forward_with_prologues_equals_two_stage(pro):
    K, N, M = 1152, 2304, 3000
    layer = _layer(K, N, 5)
    x = (torch.randn((M, K), device=DEV) * 2).half()
    sc, sh = torch.randn(K, device=DEV) * 0.1, torch.randn(K, device=DEV) * 0.1
    p = {"mod": dtq.Prologue(dtq.PROLOGUE_MODULATE, sc, sh),
         "ln": dtq.Prologue(dtq.PROLOGUE_LN_MODULATE, sc, sh, 1e-6),
         "gelu": dtq.Prologue(dtq.PROLOGUE_GELU)}[pro]
    want = _two_stage(layer, x, torch.float16, p)
    assert torch.equal(layer.forward(x, prologue=p), want)


def test_shared_workspace_mixed_m_and_graph_replay():
    # the stack's pattern: layers of different M share one workspace, back to
    # back (programmatic launches chain them), captured once and replayed
    K = 1152
    layers = [_layer(K, n, i) for i, n in enumerate((3456, 1152, 2304, 4608))]
    rows = (4096, 4096, 480, 4096)
    xs = [(torch.randn((m, K), device=DEV) * 2).half() for m in rows]
    ws = layers[3].workspace(4096, DEV)
    outs = [torch.empty((m, l.N), dtype=torch.float16, device=DEV) for m, l in zip(rows, layers)]
    want = [_two_stage(l, x, torch.float16) for l, x in zip(layers, xs)]

    def run():
        for l, x, o in zip(layers, xs, outs):
            l.forward(x, out=o, workspace=ws)

    run()
    torch.cuda.synchronize()
    for o, w in zip(outs, want):
        assert torch.equal(o, w)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run()
    for _ in range(20):
        for o in outs:
            o.zero_()
        g.replay()
        torch.cuda.synchronize()
        for o, w in zip(outs, want):
            assert torch.equal(o, w)
    assert int(ws[:8192 * 4 + 4].count_nonzero()) == 0
