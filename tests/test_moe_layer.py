"""Caller-side integration: an MoE layer on the Buffer API
(tools/moe_layer.py) equals a dense, communication-free evaluation of the same
experts — normal mode (prefill), LL FP8 mode (decode), LL with the recv hook
overlapping a shared expert, and LL replayed from a CUDA graph."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    if not t.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    return t


def _layer(torch, T=300, H=1024, Fd=256, E=16, k=4, Tm=128):
    import paper_2512_19849_b200 as epb
    from tools.moe_layer import MoELayer
    buf = epb.Buffer(None, epb.nvl_bytes_hint(T, H, 1, k), epb.Buffer.get_low_latency_rdma_size_hint(
        Tm, H, 1, E, num_topk=k), low_latency_mode=True)
    layer = MoELayer(buf, H, Fd, E, k, seed=3)
    g = torch.Generator(device="cpu").manual_seed(4)
    x = torch.randn(T, H, generator=g).to("cuda", torch.bfloat16)
    return buf, layer, x


def test_moe_layer_normal_matches_dense(torch):
    from tools.moe_layer import dense_reference
    buf, layer, x = _layer(torch)
    idx, w = layer.route(x)
    out = layer.forward_normal(x, idx, w)
    ref = dense_reference(layer, x, idx, w)
    torch.testing.assert_close(out.float(), ref.float(), rtol=2e-2, atol=2e-2)
    buf.destroy()


def test_moe_layer_ll_hook_and_graph(torch):
    import paper_2512_19849_b200 as epb
    from tools.moe_layer import dense_reference
    buf, layer, x = _layer(torch)
    Tm = 128
    xd = x[:Tm].contiguous()
    idx, w = layer.route(xd)
    out = layer.forward_ll(xd, idx, w, Tm)
    # reference on the FP8-rounded inputs the experts actually see
    q, s = epb.per_token_cast_to_fp8(xd)
    xq = (q.float().view(Tm, -1, 128) * s.unsqueeze(-1)).view(Tm, -1).to(torch.bfloat16)
    ref = dense_reference(layer, xq, idx, w)
    torch.testing.assert_close(out.float(), ref.float(), rtol=2e-2, atol=2e-2)
    # recv hook: the shared expert runs while the tokens are in flight; same output
    out2, shared = layer.forward_ll(xd, idx, w, Tm, overlap=True)
    assert torch.equal(out2, out)
    torch.testing.assert_close(shared.float(), (xd @ layer.shared).float())
    # CUDA graph replay of the whole decode layer
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            gout = layer.forward_ll(xd, idx, w, Tm)
    torch.cuda.current_stream().wait_stream(st)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(gout, out)
    buf.destroy()
