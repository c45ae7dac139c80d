"""W4A8 forward through s8 weights unpacked into the workspace
(w4_unpack_kernel + the W8A8 kernels) against the in-GEMM nibble unpack of
the standalone GEMM (`QuantLinear.gemm`): the same int32 accumulators
(qgemm.cpp:52-60, weights c - 8) and the same fp outputs bit for bit -- the
in-GEMM path folds an exact factor 16 out of s_x and the zero-point term, so
the two epilogues round identically."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import paper_2406_02540_b200 as dtq  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _layer(rng, N, K, bias=True, packed=False):
    wc = rng.integers(0, 16, (N, K), dtype=np.uint8)
    s = torch.from_numpy(rng.uniform(0.5, 2.0, N) * 1e-2).to(DEV)
    b = torch.from_numpy(rng.standard_normal(N) * 0.1).to(DEV) if bias else None
    if packed:
        wp = np.zeros((N, (K + 1) // 2), np.uint8)
        wp |= wc[:, 0::2]
        wp[:, : K // 2] |= (wc[:, 1::2] << 4).astype(np.uint8)
        return dtq.QuantLinear.from_codes(torch.from_numpy(wp).to(DEV), s, 4, K, bias=b,
                                          packed=True), wc
    return dtq.QuantLinear.from_codes(torch.from_numpy(wc).to(DEV), s, 4, K, bias=b), wc


@pytest.mark.parametrize("M,K,N", [(4096, 1152, 4608), (4096, 1152, 3456), (1000, 4608, 1152),
                                   (300, 200, 100), (77, 13, 37), (513, 328, 96)])
@pytest.mark.parametrize("out", [torch.float16, torch.float32])
def test_forward_matches_in_gemm_unpack(M, K, N, out):
    rng = np.random.default_rng(M + K + N)
    layer, wc = _layer(rng, N, K, packed=K == 328)
    x = torch.from_numpy(rng.standard_normal((M, K)).astype(np.float16)).to(DEV)
    y = layer.forward(x, out_dtype=out)
    codes, s, z = layer.quantize(x)
    assert torch.equal(y, layer.gemm(codes, s, z, out_dtype=out))
    if M * N <= 1 << 20:  # the accumulator against the reference's integer sum
        acc = layer.gemm(codes, s, z, out_dtype=torch.int32).cpu().numpy().astype(np.int64)
        a = codes.cpu().numpy().astype(np.int64) - z.cpu().numpy()[:, None]
        assert np.array_equal(acc, a @ (wc.astype(np.int64) - 8).T)


def test_gelu_epilogue_on_unpacked_weights():
    rng = np.random.default_rng(3)
    layer, _ = _layer(rng, 4608, 1152)
    x = torch.from_numpy(rng.standard_normal((2048, 1152)).astype(np.float16)).to(DEV)
    y = layer.forward(x, activation=dtq.ACT_GELU).float()
    ref = torch.nn.functional.gelu(layer.forward(x, out_dtype=torch.float32))
    err = (y - ref).abs().max() / ref.abs().max()
    assert float(err) <= 1e-3


def test_shared_workspace_back_to_back():
    # two W4 layers alternate on one workspace with no synchronisation: each
    # forward's unpack overwrites the s8 weights the previous forward's GEMM
    # reads (griddepcontrol.wait orders it), eagerly and in a CUDA graph
    rng = np.random.default_rng(11)
    M, K, N = 4096, 1152, 3456
    la, _ = _layer(rng, N, K)
    lb, _ = _layer(rng, N, K)
    xs = [torch.from_numpy(rng.standard_normal((M, K)).astype(np.float16)).to(DEV)
          for _ in range(2)]
    want = [la.forward(xs[0]), lb.forward(xs[1])]
    ws = la.workspace(M, DEV)
    outs = [torch.empty((M, N), dtype=torch.float16, device=DEV) for _ in range(6)]

    def run():
        for i in range(6):
            (la if i % 2 == 0 else lb).forward(xs[i % 2], out=outs[i], workspace=ws)

    run()
    torch.cuda.synchronize()
    for i in range(6):
        assert torch.equal(outs[i], want[i % 2]), i
    for o in outs:
        o.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    for i in range(6):
        assert torch.equal(outs[i], want[i % 2]), i


def test_workspace_size_covers_unpacked_weights():
    rng = np.random.default_rng(2)
    w4, _ = _layer(rng, 4608, 1152)
    w8 = dtq.QuantLinear.from_codes(torch.from_numpy(rng.integers(0, 256, (4608, 1152),
                                                                  dtype=np.uint8)).to(DEV),
                                    torch.ones(4608, dtype=torch.float64, device=DEV), 8, 1152)
    n4 = dtq.lib().dtq_qlinear_workspace_bytes(w4._h, 100)
    n8 = dtq.lib().dtq_qlinear_workspace_bytes(w8._h, 100)
    assert n4 - n8 == 4608 * 1152
    small = torch.zeros(n4 - 1, dtype=torch.uint8, device=DEV)
    x = torch.randn(100, 1152, device=DEV).half()
    with pytest.raises(ValueError):
        w4.forward(x, workspace=small)


def test_forward_host_pipeline_w4():
    # the host pipeline's geometric row chunks (128, 256, 512, 1024, rest)
    # share one workspace: every chunk's quantizer re-expands the weights
    rng = np.random.default_rng(8)
    layer, _ = _layer(rng, 4608, 1152)
    x = torch.from_numpy(rng.standard_normal((4096, 1152)).astype(np.float16))
    want = layer.forward(x.to(DEV)).cpu()
    xh = x.pin_memory()
    yh = torch.empty((4096, 4608), dtype=torch.float16).pin_memory()
    layer.forward_host(xh, yh)
    assert torch.equal(yh, want)


def test_unaligned_workspace_is_rejected():
    # the workspace holds TMA operands (codes; a W4A8 forward's s8 weights)
    rng = np.random.default_rng(12)
    layer, _ = _layer(rng, 1152, 1152)
    x = torch.from_numpy(rng.standard_normal((700, 1152)).astype(np.float16)).to(DEV)
    n = dtq.lib().dtq_qlinear_workspace_bytes(layer._h, 700)
    big = torch.zeros(n + 64, dtype=torch.uint8, device=DEV)
    with pytest.raises(ValueError, match="16-byte aligned"):
        layer.forward(x, workspace=big[8:8 + n])
    assert torch.equal(layer.forward(x, workspace=big[16:16 + n]), layer.forward(x))
