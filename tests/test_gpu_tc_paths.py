"""Triangle counting across the code paths of gb_tc (gb_mxm.cu) against the C
oracle (oracle/cgraph.c, pinned to the reference's counts in
test_oracle.py): graphs small enough that every rank sits in the per-warp
bitmap and the dense hub rows (n < 8,192), graphs whose low ranks take the
adjacency-search fallback (n > 32,768), rows longer than the 2,048-entry
tile of the upper-row build, hubs whose dense rows need more than the 32-word
top window, and graphs with no triangles at all."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gb():
    import paper_1908_01407_b200 as gb
    return gb


def _sym(gb, r, c, n):
    keep = r != c
    r, c = r[keep], c[keep]
    rr, cc = np.r_[r, c], np.r_[c, r]
    return gb.SparseMatrix.from_tuples(rr, cc, np.ones(rr.size, np.int64), n, n,
                                       dedup=gb.builtin_monoid("LogicalOr"))


def _oracle(A):
    from oracle import cgraph
    o = A.orient(False)
    return cgraph.tc(o.offsets.cpu().numpy(), o.indices.cpu().numpy())


@pytest.mark.parametrize("n,m,seed", [(40, 200, 1), (3000, 40000, 2), (20000, 300000, 3),
                                      (50000, 600000, 4), (120000, 900000, 5)])
def test_tc_uniform_random(gb, n, m, seed):
    rng = np.random.default_rng(seed)
    A = _sym(gb, rng.integers(0, n, m), rng.integers(0, n, m), n)
    assert gb.triangle_count(A) == _oracle(A)


@pytest.mark.parametrize("scale", [10, 13, 15, 17])
def test_tc_rmat(gb, scale):
    A = gb.io.rmat_matrix(scale)
    assert gb.triangle_count(A) == _oracle(A)


@pytest.mark.parametrize("n_hubs,n", [(3, 10000), (40, 60000)])
def test_tc_hubs_and_cliques(gb, n_hubs, n):
    """A few hubs adjacent to everything (rows far above the 2,048-entry tile,
    dense rows spanning the whole top range) over a sparse random rest plus
    small cliques."""
    rng = np.random.default_rng(n_hubs)
    r, c = [], []
    for h in range(n_hubs):
        r.append(np.full(n - 1, h))
        c.append(np.delete(np.arange(n), h))
    m = 4 * n
    r.append(rng.integers(0, n, m))
    c.append(rng.integers(0, n, m))
    for base in range(n_hubs, n_hubs + 200, 10):   # 20 cliques of 10
        ids = np.arange(base, base + 10)
        a, b = np.meshgrid(ids, ids)
        r.append(a.ravel())
        c.append(b.ravel())
    A = _sym(gb, np.concatenate(r), np.concatenate(c), n)
    assert gb.triangle_count(A) == _oracle(A)


def test_tc_triangle_free(gb):
    """A bipartite graph and a long cycle: no triangles on any path."""
    n = 40000
    rng = np.random.default_rng(9)
    r = rng.integers(0, n // 2, 200000)
    c = rng.integers(n // 2, n, 200000)
    assert gb.triangle_count(_sym(gb, r, c, n)) == 0
    i = np.arange(n)
    assert gb.triangle_count(_sym(gb, i, (i + 1) % n, n)) == 0
