"""GPU parity of the network runtime (include/lcnn_net.h) against the
UNMODIFIED reference run_network (net.cpp:266-398, via oracle/_ref):
same JSON, same (c_t, n_t) annotation, same seeded default weights
(net.cpp:217-243), same input.

Tolerances:
  FP32 dense precision : approx_equal 1e-5 -- the reference's own bar for
                         layout independence (test_net.cpp:211-248,
                         acceptance.cpp:328-401);
  TF32 dense precision : |p - p_ref| <= 2e-3 absolute on the softmax
                         probabilities (tf32 operand truncation, 2^-9 relative
                         per product, through three fc layers).
The pipelined host-buffer API (lcnn_net_forward_host_many) must return exactly
what the device-buffer forward returns (FP32 is deterministic).
"""
import json

import numpy as np
import pytest

from oracle.oracle import CHWN, NCHW, Ref, approx_equal, rng_uniform
from paper_1610_03618_b200 import capi, netapi

pytestmark = pytest.mark.gpu

# AlexNet's layer kinds and filter/stride pattern at a size the CPU reference
# finishes in seconds (conv1 f11 s4, overlapping 3/2 max pools, 5x5 and 3x3
# convs, two fc layers, softmax)
MINI = {
    "input": {"n": 32, "c": 3, "h": 67, "w": 67},
    "layers": [
        {"name": "conv1", "kind": "conv", "c_out": 32, "f": 11, "stride": 4, "pad": 0},
        {"name": "pool1", "kind": "pool", "win": 3, "stride": 2, "mode": "max"},
        {"name": "conv2", "kind": "conv", "c_out": 64, "f": 5, "stride": 1, "pad": 2},
        {"name": "pool2", "kind": "pool", "win": 3, "stride": 2, "mode": "avg"},
        {"name": "conv3", "kind": "conv", "c_out": 64, "f": 3, "stride": 1, "pad": 1},
        {"name": "fc6", "kind": "fc", "out": 256},
        {"name": "fc7", "kind": "fc", "out": 10},
        {"name": "prob", "kind": "softmax"},
    ],
}
THRESHOLDS = [(257, 32), (32, 128)]  # B200 calibration (all CHWN), titan-black preset (mixed)


def _nets(text, c_t, n_t):
    net = netapi.Network(text, c_t, n_t, seed=42)
    return net, net.info(NCHW)


@pytest.fixture(autouse=True)
def _restore_precision():
    yield
    netapi.set_dense_precision(capi.PREC_FP32)


@pytest.mark.parametrize("c_t,n_t", THRESHOLDS)
@pytest.mark.parametrize("precision", ["fp32", "tf32"])
def test_network_matches_reference(cuda, c_t, n_t, precision):
    import torch

    if not Ref.available():
        pytest.fail("oracle/_ref/liblcnn_ref.so missing (build() makes it)")
    text = json.dumps(MINI)
    netapi.set_dense_precision(capi.PREC_FP32 if precision == "fp32" else capi.PREC_TF32)
    net, info = _nets(text, c_t, n_t)
    rows, cols = info["out"]
    n, c, h, w = info["dims"]
    x = rng_uniform(11, n * c * h * w)
    want = Ref.run_network(text, x, NCHW, c_t, n_t, seed=42)
    assert want.shape == (rows, cols)
    # layouts: the same annotation as the reference
    ref_layouts, _ = Ref.plan_network(text, c_t, n_t)
    assert net.layouts[:len(MINI["layers"])] == ref_layouts[:len(MINI["layers"])]
    dx = torch.from_numpy(x).to(cuda)
    dy = torch.empty(rows * cols, device=cuda)
    stream = torch.cuda.current_stream(cuda).cuda_stream
    net.forward(dx.data_ptr(), NCHW, dy.data_ptr(), stream)
    torch.cuda.synchronize()
    got = dy.cpu().numpy().reshape(rows, cols)
    if precision == "fp32":
        assert approx_equal(got, want, 1e-5)
    else:
        assert np.abs(got - want).max() <= 2e-3
    assert np.allclose(got.sum(1), 1.0, atol=1e-5)
    net.close()


@pytest.mark.parametrize("c_t,n_t", THRESHOLDS)
def test_forward_host_many_matches_device_forward(cuda, c_t, n_t):
    import torch

    netapi.set_dense_precision(capi.PREC_FP32)
    net, info = _nets(json.dumps(MINI), c_t, n_t)
    rows, cols = info["out"]
    n, c, h, w = info["dims"]
    batches = [rng_uniform(100 + i, n * c * h * w) for i in range(5)]
    stream = torch.cuda.current_stream(cuda).cuda_stream
    want = []
    for b in batches:
        dy = torch.empty(rows * cols, device=cuda)
        net.forward(torch.from_numpy(b).to(cuda).data_ptr(), NCHW, dy.data_ptr(), stream)
        torch.cuda.synchronize()
        want.append(dy.cpu().numpy())
    hx = [torch.from_numpy(b).pin_memory() for b in batches]
    hy = [torch.zeros(rows * cols).pin_memory() for _ in batches]
    net.forward_host_many([t.data_ptr() for t in hx], NCHW, [t.data_ptr() for t in hy])
    for got, exp in zip(hy, want):
        assert np.array_equal(got.numpy(), exp)
    # a single batch and an empty sequence
    one = torch.zeros(rows * cols).pin_memory()
    net.forward_host_many([hx[3].data_ptr()], NCHW, [one.data_ptr()])
    assert np.array_equal(one.numpy(), want[3])
    net.forward_host_many([], NCHW, [])
    # forward_host (one batch) agrees too, in the other input layout
    xc = np.ascontiguousarray(batches[2].reshape(n, c, h, w).transpose(1, 2, 3, 0)).ravel()
    hc = torch.from_numpy(xc).pin_memory()
    out = torch.zeros(rows * cols).pin_memory()
    net.forward_host(hc.data_ptr(), CHWN, out.data_ptr())
    assert approx_equal(out.numpy(), want[2], 1e-5)
    net.close()


def test_nonfinite_input_surfaces_domain_error(cuda):
    """The reference raises DomainError for a non-finite classifier input
    (softmax.cpp:15-19, rewrapped with the layer name by net.cpp:387-391).
    Device forward: asynchronous, the sticky flag is reported by status();
    host-buffer forwards: LCNN_EDOMAIN directly."""
    import torch

    from paper_1610_03618_b200.errors import DomainError

    net = netapi.Network(json.dumps(MINI), 257, 32, seed=42, precision=capi.PREC_FP32)
    info = net.info(NCHW)
    rows, cols = info["out"]
    n, c, h, w = info["dims"]
    x = rng_uniform(5, n * c * h * w)
    bad = x.copy()
    bad[123] = np.inf
    stream = torch.cuda.current_stream(cuda).cuda_stream
    dy = torch.empty(rows * cols, device=cuda)
    net.forward(torch.from_numpy(x).to(cuda).data_ptr(), NCHW, dy.data_ptr(), stream)
    net.status(stream)  # finite: no error
    net.forward(torch.from_numpy(bad).to(cuda).data_ptr(), NCHW, dy.data_ptr(), stream)
    with pytest.raises(DomainError, match="layer 'prob': softmax: non-finite input"):
        net.status(stream)
    net.status(stream)  # the flag was cleared by the read
    out = torch.zeros(rows * cols).pin_memory()
    with pytest.raises(DomainError):
        net.forward_host(torch.from_numpy(bad).pin_memory().data_ptr(), NCHW, out.data_ptr())
    net.forward_host(torch.from_numpy(x).pin_memory().data_ptr(), NCHW, out.data_ptr())
    net.close()


def test_precision_is_per_network(cuda):
    """Two networks at different precisions side by side (and the process
    default changed in between) each keep the precision they were made with."""
    import threading

    import torch

    text = json.dumps(MINI)
    n, c, h, w = MINI["input"]["n"], 3, 67, 67
    x = torch.from_numpy(rng_uniform(9, n * c * h * w)).to(cuda)
    nets = {p: netapi.Network(text, 257, 32, seed=42, precision=p)
            for p in (capi.PREC_FP32, capi.PREC_TF32)}
    netapi.set_dense_precision(capi.PREC_TF32)  # must not affect the FP32 network
    want = {}
    for p, net in nets.items():
        assert net.precision == p
        y = torch.empty(n * 10, device=cuda)
        net.forward(x.data_ptr(), NCHW, y.data_ptr(), torch.cuda.current_stream(cuda).cuda_stream)
        torch.cuda.synchronize()
        want[p] = y.cpu()
    assert not torch.equal(want[capi.PREC_FP32], want[capi.PREC_TF32])
    got, errs = {}, []

    def run(p):
        try:
            s = torch.cuda.Stream(cuda)
            y = torch.empty(n * 10, device=cuda)
            for _ in range(20):
                nets[p].forward(x.data_ptr(), NCHW, y.data_ptr(), s.cuda_stream)
            s.synchronize()
            got[p] = y.cpu()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ts = [threading.Thread(target=run, args=(p,)) for p in nets]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    assert torch.equal(got[capi.PREC_FP32], want[capi.PREC_FP32])
    assert torch.allclose(got[capi.PREC_TF32], want[capi.PREC_TF32], rtol=1e-4, atol=1e-7)
    for net in nets.values():
        net.close()


def test_network_runs_tuned_pool_plans(cuda):
    """Every pooling layer of a Network is tuned at creation (lcnn_pool_tune;
    lcnn_net_pool_plan reports it) and the forward that runs those plans
    still matches the reference run_network (pool.cpp tap order is kept)."""
    import torch

    text = json.dumps(MINI)
    net = netapi.Network(text, 257, 32, seed=42, precision=capi.PREC_FP32)
    plans = net.pool_plans()
    pool_layers = [i for i, L in enumerate(MINI["layers"]) if L["kind"] == "pool"]
    assert sorted(plans) == pool_layers and all(p.tuned == 1 for p in plans.values())
    info = net.info(NCHW)
    rows, cols = info["out"]
    n, c, h, w = info["dims"]
    x = rng_uniform(21, n * c * h * w)
    dy = torch.empty(rows * cols, device=cuda)
    net.forward(torch.from_numpy(x).to(cuda).data_ptr(), NCHW, dy.data_ptr(),
                torch.cuda.current_stream(cuda).cuda_stream)
    torch.cuda.synchronize()
    want = Ref.run_network(text, x, NCHW, 257, 32, seed=42)
    assert approx_equal(dy.cpu().numpy().reshape(rows, cols), want, 1e-5)
    net.close()


def test_forward_concurrent_streams_and_graph_replay_agree(cuda):
    """In-kernel stream-K zeroing keeps per-stream / per-capture sync words
    (Network::sync_words): forwards on two streams at once, and a captured
    CUDA graph replayed on a third stream while a stream forward runs, give
    the single-stream logits.  AlexNet at batch 128, TF32: conv4 / conv5 /
    fc6 / fc7 all have stream-K tails (the in-kernel zeroing path)."""
    import os

    import torch

    text = open(os.path.join(os.path.dirname(__file__), "..", "configs", "alexnet.json")).read()
    net = netapi.Network(text, 257, 32, seed=42, precision=capi.PREC_TF32)
    info = net.info(NCHW)
    rows, cols = info["out"]
    dn, dc, dh, dw = info["dims"]
    g = torch.Generator(device=cuda).manual_seed(5)
    x = torch.rand(dn * dc * dh * dw, device=cuda, generator=g) * 2 - 1
    lay = info["first_layout"]
    main = torch.cuda.current_stream(cuda)
    ref = torch.empty(rows * cols, device=cuda)
    net.forward(x.data_ptr(), lay, ref.data_ptr(), main.cuda_stream)
    torch.cuda.synchronize()
    s1, s2, s3 = (torch.cuda.Stream(cuda) for _ in range(3))
    y1 = torch.empty_like(ref)
    y2 = torch.empty_like(ref)
    for _ in range(4):
        y1.fill_(float("nan"))
        y2.fill_(float("nan"))
        torch.cuda.synchronize()
        net.forward(x.data_ptr(), lay, y1.data_ptr(), s1.cuda_stream)
        net.forward(x.data_ptr(), lay, y2.data_ptr(), s2.cuda_stream)
        torch.cuda.synchronize()
        assert torch.allclose(y1, ref, rtol=1e-4, atol=1e-7)
        assert torch.allclose(y2, ref, rtol=1e-4, atol=1e-7)
    yg = torch.empty_like(ref)
    graph = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream(cuda)
    cap.wait_stream(main)
    with torch.cuda.graph(graph, stream=cap):
        net.forward(x.data_ptr(), lay, yg.data_ptr(), cap.cuda_stream)
    torch.cuda.synchronize()
    for _ in range(4):
        yg.fill_(float("nan"))
        y1.fill_(float("nan"))
        torch.cuda.synchronize()
        with torch.cuda.stream(s3):
            graph.replay()
        net.forward(x.data_ptr(), lay, y1.data_ptr(), s1.cuda_stream)
        torch.cuda.synchronize()
        assert torch.allclose(yg, ref, rtol=1e-4, atol=1e-7)
        assert torch.allclose(y1, ref, rtol=1e-4, atol=1e-7)
    net.close()


def test_forward_graph_replays_match_the_stream_forward(cuda):
    """lcnn_net_forward_graph: captured once per buffer triple, replayed after;
    the logits match lcnn_net_forward (TF32 AlexNet: stream-K tails, fused
    conv1+pool1, in-kernel zeroing all inside the graph), a second buffer
    pair gets its own graph, and a non-finite input still raises through
    lcnn_net_status."""
    import os

    import torch

    text = open(os.path.join(os.path.dirname(__file__), "..", "configs", "alexnet.json")).read()
    net = netapi.Network(text, 257, 32, seed=42, precision=capi.PREC_TF32)
    info = net.info(NCHW)
    rows, cols = info["out"]
    dn, dc, dh, dw = info["dims"]
    lay = info["first_layout"]
    g = torch.Generator(device=cuda).manual_seed(11)
    xs = [torch.rand(dn * dc * dh * dw, device=cuda, generator=g) * 2 - 1 for _ in range(2)]
    s = torch.cuda.current_stream(cuda).cuda_stream
    refs = []
    for x in xs:
        r = torch.empty(rows * cols, device=cuda)
        net.forward(x.data_ptr(), lay, r.data_ptr(), s)
        refs.append(r)
    ys = [torch.empty(rows * cols, device=cuda) for _ in xs]
    for _ in range(3):
        for x, y, r in zip(xs, ys, refs):
            y.fill_(float("nan"))
            net.forward_graph(x.data_ptr(), lay, y.data_ptr(), s)
            torch.cuda.synchronize()
            assert torch.allclose(y, r, rtol=1e-4, atol=1e-7)
    # new input values in the same buffer: the replay reads them
    xs[0].mul_(0.5)
    net.forward(xs[0].data_ptr(), lay, refs[0].data_ptr(), s)
    net.forward_graph(xs[0].data_ptr(), lay, ys[0].data_ptr(), s)
    torch.cuda.synchronize()
    assert torch.allclose(ys[0], refs[0], rtol=1e-4, atol=1e-7)
    net.status(s)
    xs[1][0] = float("inf")
    net.forward_graph(xs[1].data_ptr(), lay, ys[1].data_ptr(), s)
    with pytest.raises(Exception):
        net.status(s)
    net.close()


def test_forward_graph_cache_eviction_and_many_captures(cuda):
    """More buffer pairs than the graph cache holds (16) and than the spare
    sync-word sets (8): later captures run with zeroing launches instead of
    in-kernel zeroing, the oldest graph is evicted and re-captured on reuse,
    and every replay still matches the stream forward."""
    import json as _json

    import torch

    net = netapi.Network(_json.dumps(MINI), 257, 32, seed=42, precision=capi.PREC_TF32)
    info = net.info(NCHW)
    rows, cols = info["out"]
    dn, dc, dh, dw = info["dims"]
    lay = info["first_layout"]
    g = torch.Generator(device=cuda).manual_seed(3)
    x = torch.rand(dn * dc * dh * dw, device=cuda, generator=g) * 2 - 1
    s = torch.cuda.current_stream(cuda).cuda_stream
    ref = torch.empty(rows * cols, device=cuda)
    net.forward(x.data_ptr(), lay, ref.data_ptr(), s)
    outs = [torch.empty(rows * cols, device=cuda) for _ in range(20)]
    for rep in range(2):
        for y in outs:
            y.fill_(float("nan"))
            net.forward_graph(x.data_ptr(), lay, y.data_ptr(), s)
        torch.cuda.synchronize()
        for y in outs:
            assert torch.allclose(y, ref, rtol=1e-4, atol=1e-7), rep
    net.close()
