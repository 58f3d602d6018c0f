"""Calls issued under different torch streams (gb_ctx follows the current
stream; a switch orders the new stream after the previous one): asynchronous
bfs calls alternating between streams, the device loops and a masked pull on
a side stream -- results equal the same calls on the default stream."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gb():
    import paper_1908_01407_b200 as gb
    return gb


def test_async_bfs_alternating_streams(gb):
    A = gb.io.rmat_matrix(14)
    B = gb.io.rmat_matrix(13, a=.25, b=.25, c=.25, d=.25)
    srcs = [0, 5, 17, 1, 2, 99]
    want = {(g, s): gb.bfs(G, s).values for g, G in (("A", A), ("B", B)) for s in srcs}
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = []
    for i, s in enumerate(srcs * 3):
        name, G = ("A", A) if i % 3 else ("B", B)
        with torch.cuda.stream(streams[i % 2]):
            d = gb.Descriptor()
            outs.append((name, s, gb.bfs(G, s, desc=d), d))
    torch.cuda.synchronize()
    for name, s, lv, d in outs:
        assert np.array_equal(lv.values, want[(name, s)])
        assert len(d.direction_log) >= 1


def test_loops_and_mxv_on_a_side_stream(gb):
    A = gb.io.rmat_matrix(12)
    W = gb.io.rmat_matrix(12, weighted=True)
    ref = (gb.sssp(W, 0).values, gb.pagerank(A, eps=1e-300, max_iters=10).values,
           gb.connected_components(A).values)
    n = A.nrows
    x = gb.Vector.dense_of(np.arange(n, dtype=np.float64), 0.0)
    m = gb.Vector.dense_of((np.arange(n) % 2).astype(np.int64), 0)
    d0 = gb.Descriptor(direction=gb.Direction.FORCE_PULL, mask_mode=gb.MaskMode.COMPLEMENT)
    w0 = gb.mxv(gb.builtin_semiring("PlusMultiplies"), A, x, mask=m, desc=d0).to_dense(0.0).values
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        got = (gb.sssp(W, 0).values, gb.pagerank(A, eps=1e-300, max_iters=10).values,
               gb.connected_components(A).values)
        d1 = gb.Descriptor(direction=gb.Direction.FORCE_PULL, mask_mode=gb.MaskMode.COMPLEMENT)
        w1 = gb.mxv(gb.builtin_semiring("PlusMultiplies"), A, x, mask=m, desc=d1)
    side.synchronize()
    assert np.array_equal(got[0], ref[0]) and np.array_equal(got[2], ref[2])
    assert np.abs(got[1] - ref[1]).sum() <= 1e-12
    np.testing.assert_allclose(w1.to_dense(0.0).values, w0, rtol=1e-12, atol=0)
