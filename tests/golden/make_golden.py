"""Generate the golden fixtures under tests/golden/ by running the REAL reference.

This script is the only place the read-only reference package
(/root/reference/pkg/src/graphalg) is executed.  It runs here, in the build
container, never on the GPU box; its outputs are small JSON / npz fixtures
committed next to it.  Usage::

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--big]

``--big`` additionally runs the scale-20 algorithm goldens (minutes each; the
TC s20 run takes ~9 minutes single-threaded in the reference).

Fixtures written:
  rmat_graphs.json     CSR digests (and nnz/levels) of reference-generated RMAT graphs
  rmat_s10.npz         full CSR + weights of the s10 graph (bit-exact generator check)
  algorithms.json      bfs/sssp/pagerank/cc/tc outputs (digests, traces, counts)
  kernel_cases.json    seeded kernel instances: inputs + reference outputs + counters
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

sys.dont_write_bytecode = True
sys.path.insert(0, REF_SRC)
import graphalg as ref  # noqa: E402  (the reference, read-only)
from graphalg import cli as ref_cli  # noqa: E402


def csr_digest(A):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(A.row_offsets, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(A.col_indices, dtype=np.int64).tobytes())
    return h.hexdigest()


def values_digest(vals):
    return hashlib.sha256(np.ascontiguousarray(vals, dtype=np.float64).tobytes()).hexdigest()


def build(scale, weighted=False, ef=16, a=0.57, b=0.19, c=0.19, d=0.05, seed=1):
    p = ref.RmatParams(scale=scale, edge_factor=ef, a=a, b=b, c=c, d=d, seed=seed)
    e = ref.preprocess(ref.generate_rmat(p), make_undirected=True)
    if weighted:
        e = ref.assign_weights(e, 1, 64, seed=seed)
    return ref.edges_to_matrix(e, weighted=weighted)


def trace_of(desc):
    return [[dd.chosen, int(dd.frontier_nvals), int(dd.estimated_frontier_edges),
             float(dd.threshold_edges)] for dd in desc.direction_log]


# ---------------------------------------------------------------------------
# graphs
# ---------------------------------------------------------------------------

def make_graphs(out, scales):
    graphs = {}
    for name, kw in [("rmat", {}), ("uniform", dict(a=0.25, b=0.25, c=0.25, d=0.25))]:
        for s in scales:
            if name == "uniform" and s > 14:
                continue
            t = time.time()
            A = build(s, **kw)
            W = build(s, weighted=True, **kw) if s <= 14 else None
            key = f"{name}_s{s}"
            graphs[key] = dict(scale=s, n=A.nrows, nnz=A.nnz, csr=csr_digest(A),
                               max_deg=int(np.diff(A.row_offsets).max()),
                               weights=None if W is None else values_digest(W.csr_values))
            print(f"graph {key}: nnz={A.nnz} ({time.time()-t:.1f}s)", flush=True)
            if key == "rmat_s10":
                Wf = build(10, weighted=True)
                np.savez_compressed(os.path.join(HERE, "rmat_s10.npz"),
                                    row_offsets=A.row_offsets, col_indices=A.col_indices,
                                    weights=Wf.csr_values)
    out["graphs"] = graphs


# ---------------------------------------------------------------------------
# algorithms
# ---------------------------------------------------------------------------

def run_algorithms(scales_bfs, scales_other, big):
    res = {}
    for s in scales_bfs:
        A = build(s)
        desc = ref.Descriptor()
        t = time.time()
        lv = ref.bfs(A, 0, desc=desc)
        res[f"bfs_s{s}"] = dict(digest=ref_cli._digest(lv), trace=trace_of(desc),
                                reached=int(np.count_nonzero(lv.values)),
                                levels=int(lv.values.max()),
                                level_counts=np.bincount(lv.values).tolist())
        if s <= 12:
            res[f"bfs_s{s}"]["values"] = lv.values.tolist()
        print(f"bfs s{s} {time.time()-t:.1f}s", flush=True)
        # a second source (a mid-degree vertex) exercises other traces
        src = int(np.argsort(np.diff(A.row_offsets), kind="stable")[A.nrows // 2 + A.nrows // 4])
        desc = ref.Descriptor()
        lv = ref.bfs(A, src, desc=desc)
        res[f"bfs_s{s}_src{src}"] = dict(source=src, digest=ref_cli._digest(lv), trace=trace_of(desc))
    for s in scales_other:
        W = build(s, weighted=True)
        desc = ref.Descriptor()
        t = time.time()
        iters = []
        dist = ref.sssp(W, 0, desc=desc, on_iteration=lambda it, d: iters.append(it))
        res[f"sssp_s{s}"] = dict(digest=ref_cli._digest(dist), trace=trace_of(desc),
                                 iterations=len(iters),
                                 finite=int(np.isfinite(dist.values).sum()))
        if s <= 12:
            res[f"sssp_s{s}"]["values"] = [float(x) for x in dist.values]
        print(f"sssp s{s} {time.time()-t:.1f}s", flush=True)

        A = build(s)
        t = time.time()
        desc = ref.Descriptor()
        cc = ref.connected_components(A, desc=desc)
        res[f"cc_s{s}"] = dict(digest=ref_cli._digest(cc), trace=trace_of(desc),
                               components=int(np.unique(cc.values).size))
        if s <= 12:
            res[f"cc_s{s}"]["values"] = cc.values.tolist()
        print(f"cc s{s} {time.time()-t:.1f}s", flush=True)

        t = time.time()
        pr = ref.pagerank(A, alpha=0.85, eps=1e-300, max_iters=20)
        pr_default = ref.pagerank(A)
        res[f"pr_s{s}"] = dict(sum=float(pr.values.sum()), l1_first_last=None,
                               sum_default=float(pr_default.values.sum()),
                               digest9=ref_cli._digest(pr))
        if s <= 14:
            np.save(os.path.join(HERE, f"pr_s{s}.npy"), pr.values)
            np.save(os.path.join(HERE, f"pr_default_s{s}.npy"), pr_default.values)
        print(f"pr s{s} {time.time()-t:.1f}s", flush=True)

        if s <= 14 or big:
            t = time.time()
            tc = ref.triangle_count(A)
            res[f"tc_s{s}"] = dict(count=int(tc))
            print(f"tc s{s} = {tc} {time.time()-t:.1f}s", flush=True)
    # uniform graph family
    for s in (10, 12):
        A = build(s, a=0.25, b=0.25, c=0.25, d=0.25)
        desc = ref.Descriptor()
        lv = ref.bfs(A, 0, desc=desc)
        cc = ref.connected_components(A)
        res[f"uniform_bfs_s{s}"] = dict(digest=ref_cli._digest(lv), trace=trace_of(desc))
        res[f"uniform_cc_s{s}"] = dict(digest=ref_cli._digest(cc))
        res[f"uniform_tc_s{s}"] = dict(count=int(ref.triangle_count(A)))
    return res


# ---------------------------------------------------------------------------
# kernel-level cases
# ---------------------------------------------------------------------------

def rand_matrix(rng, nr, nc, density, dtype, low, high, build_csc=True):
    stored = rng.random((nr, nc)) < density
    r, c = np.nonzero(stored)
    if np.dtype(dtype).kind == "i":
        v = rng.integers(low, high + 1, size=r.size).astype(dtype)
    else:
        v = (rng.random(r.size) * (high - low) + low).astype(dtype)
    return ref.SparseMatrix.from_tuples(r, c, v, nr, nc, build_csc=build_csc)


def rand_vector(rng, n, k, dtype, low, high, dense=False, zero=None):
    k = min(k, n)
    idx = np.sort(rng.choice(n, size=k, replace=False)) if k else np.empty(0, np.int64)
    if np.dtype(dtype).kind == "i":
        vals = rng.integers(low, high + 1, size=k).astype(dtype)
    else:
        vals = (rng.random(k) * (high - low) + low).astype(dtype)
    v = ref.Vector.from_entries(idx, vals, n, dtype=dtype)
    if dense:
        v = v.to_dense(zero if zero is not None else 0)
    return v


def rand_mask(rng, n, dense):
    if dense:
        return ref.Vector.dense_of((rng.random(n) < 0.5).astype(np.int64), 0)
    idx = np.flatnonzero(rng.random(n) < 0.5)
    vals = (rng.random(idx.size) < 0.8).astype(np.int64)
    return ref.Vector.from_entries(idx, vals, n)


def vec_json(v):
    if v is None:
        return None
    return dict(size=v.size, sparse=v.is_sparse,
                indices=None if v.indices is None else v.indices.tolist(),
                values=[x.item() for x in np.asarray(v.values)],
                dtype=str(v.values.dtype), zero=np.asarray(v.zero).item())


def mat_json(A):
    r, c, v = A.extract_tuples()
    return dict(nrows=A.nrows, ncols=A.ncols, rows=r.tolist(), cols=c.tolist(),
                values=[x.item() for x in v], dtype=str(A.dtype), has_csc=A.has_csc)


def counters_json(desc):
    c = desc.counters
    return [c.matrix_entries_read, c.semiring_multiplies, c.semiring_adds]


SEMIRINGS = ["PlusMultiplies", "LogicalOrAnd", "MinPlus", "MaxPlus", "MinMultiplies",
             "MinimumSelectSecond", "PlusLess", "MinimumNotEqualTo"]


def make_desc(mode, transpose_attr=None, direction="auto", early=False, workers=1, partition="nonzero"):
    d = ref.Descriptor()
    if mode == "complement":
        d.toggle("mask")
    if transpose_attr:
        d.toggle(transpose_attr)
    d.direction = ref.Direction(direction)
    d.early_exit = early
    d.num_workers = workers
    d.partition = ref.Partition(partition)
    return d


def kernel_cases(seed=20240917):
    rng = np.random.default_rng(seed)
    cases = []

    def add(kind, **kw):
        kw["kind"] = kind
        cases.append(kw)

    # matrix-vector family
    for name in SEMIRINGS:
        sr = ref.builtin_semiring(name)
        dtypes = [np.int64] if name in ("LogicalOrAnd", "MinimumSelectSecond",
                                         "MinimumNotEqualTo") else [np.int64, np.float64]
        for dtype in dtypes:
            for trial in range(6):
                nr = int(rng.integers(1, 24))
                nc = nr if trial % 2 == 0 else int(rng.integers(1, 24))
                lo, hi = (0, 1) if name == "LogicalOrAnd" else (1, 9)
                A = rand_matrix(rng, nr, nc, float(rng.uniform(0.05, 0.6)), dtype, lo, hi)
                for op in ("mxv", "vxm", "pull", "push"):
                    for transpose in (False, True):
                        in_size = (nr if transpose else nc) if op in ("mxv", "pull", "push") else \
                            (nc if transpose else nr)
                        out_size = (nc if transpose else nr) if op in ("mxv", "pull", "push") else \
                            (nr if transpose else nc)
                        for mode in ("none", "normal", "complement"):
                            k = int(rng.integers(0, in_size + 1))
                            u = rand_vector(rng, in_size, k, dtype, 1, 1 if name == "LogicalOrAnd" else 9,
                                            dense=(op == "pull") or (op != "push" and rng.random() < 0.4),
                                            zero=None)
                            if op == "pull":
                                ident = sr.add.identity_for(np.result_type(A.csr_values, u.values))
                                u = rand_vector(rng, in_size, k, dtype, 1, 1 if name == "LogicalOrAnd" else 9).to_dense(ident)
                            mask = None if mode == "none" else rand_mask(rng, out_size, bool(rng.random() < 0.5))
                            direction = ["auto", "force-push", "force-pull"][int(rng.integers(0, 3))]
                            early = bool(rng.random() < 0.5)
                            if op in ("mxv", "pull", "push"):
                                tattr = "inp0" if transpose else None
                            else:
                                tattr = "inp1" if transpose else None
                            desc = make_desc(mode, tattr, direction, early)
                            try:
                                if op == "mxv":
                                    w = ref.mxv(sr, A, u, mask=mask, desc=desc)
                                elif op == "vxm":
                                    w = ref.vxm(sr, u, A, mask=mask, desc=desc)
                                elif op == "pull":
                                    w = ref.spmv_pull(sr, A, u, mask=mask, desc=desc)
                                else:
                                    w = ref.spmspv_push(sr, A, u, mask=mask, desc=desc)
                                err = None
                            except Exception as exc:  # shape mismatches etc. are goldens too
                                w, err = None, type(exc).__name__
                            add("mv", op=op, semiring=name, A=mat_json(A), u=vec_json(u),
                                mask=vec_json(mask), mask_mode=mode, transpose=transpose,
                                direction=direction, early_exit=early,
                                out=vec_json(w), error=err, counters=counters_json(desc),
                                log=[[x.chosen, x.frontier_nvals, x.estimated_frontier_edges,
                                      x.threshold_edges] for x in desc.direction_log])

    # masked SpGEMM
    for trial in range(30):
        n = int(rng.integers(1, 14))
        dtype = [np.int64, np.float64][trial % 2]
        name = ["PlusMultiplies", "MinPlus", "MaxPlus", "LogicalOrAnd", "PlusLess"][trial % 5]
        sr = ref.builtin_semiring(name)
        lo, hi = (0, 1) if name == "LogicalOrAnd" else (1, 5)
        A = rand_matrix(rng, n, n, float(rng.uniform(0.1, 0.6)), dtype, lo, hi)
        B = rand_matrix(rng, n, n, float(rng.uniform(0.1, 0.6)), dtype, lo, hi)
        M = rand_matrix(rng, n, n, float(rng.uniform(0.1, 0.6)), np.int64, 0, 1)
        tb = bool(trial % 3 == 0)
        desc = make_desc("none", "inp1" if tb else None)
        C = ref.mxm_masked(sr, A, B, mask=M, desc=desc)
        add("mxm", semiring=name, A=mat_json(A), B=mat_json(B), M=mat_json(M),
            transpose_b=tb, out=mat_json(C), counters=counters_json(desc))

    # elementwise / assign / scatter / gather / apply / reduce
    ops = {"Plus": ref.algebra.PLUS, "Minus": ref.algebra.MINUS, "Multiplies": ref.algebra.TIMES,
           "Minimum": ref.algebra.MIN, "Maximum": ref.algebra.MAX, "Less": ref.algebra.LESS,
           "NotEqualTo": ref.algebra.NOT_EQUAL, "LogicalOr": ref.algebra.LOGICAL_OR,
           "LogicalAnd": ref.algebra.LOGICAL_AND, "SelectSecond": ref.algebra.SECOND}
    for trial in range(160):
        n = int(rng.integers(1, 30))
        dtype = [np.int64, np.float64][int(rng.integers(0, 2))]
        u = rand_vector(rng, n, int(rng.integers(0, n + 1)), dtype, -5, 9, dense=bool(rng.random() < 0.5))
        v = rand_vector(rng, n, int(rng.integers(0, n + 1)), dtype, -5, 9, dense=bool(rng.random() < 0.5))
        mode = ["none", "normal", "complement"][int(rng.integers(0, 3))]
        mask = None if mode == "none" else rand_mask(rng, n, bool(rng.random() < 0.5))
        # operator: a semiring, a monoid or a bare op
        pick = int(rng.integers(0, 3))
        if pick == 0:
            opname = SEMIRINGS[int(rng.integers(0, len(SEMIRINGS)))]
            op = ref.builtin_semiring(opname)
            opkind = "semiring"
        elif pick == 1:
            opname = ["Plus", "Multiplies", "Minimum", "Maximum", "LogicalOr", "LogicalAnd"][int(rng.integers(0, 6))]
            op = ref.builtin_monoid(opname)
            opkind = "monoid"
        else:
            opname = list(ops)[int(rng.integers(0, len(ops)))]
            op = ops[opname]
            opkind = "op"
        which = ["add", "mult", "add_scalar"][trial % 3]
        desc = make_desc(mode)
        scalar = float(rng.integers(-3, 4)) if dtype == np.float64 else int(rng.integers(-3, 4))
        try:
            if which == "add":
                w = ref.ewise_add(op, u, v, mask=mask, desc=desc)
            elif which == "mult":
                w = ref.ewise_mult(op, u, v, mask=mask, desc=desc)
            else:
                w = ref.ewise_add(op, u, scalar, mask=mask, desc=desc)
            err = None
        except Exception as exc:
            w, err = None, type(exc).__name__
        add("ewise", which=which, opkind=opkind, op=opname, u=vec_json(u), v=vec_json(v),
            scalar=scalar, mask=vec_json(mask), mask_mode=mode, out=vec_json(w), error=err)

    for trial in range(60):
        n = int(rng.integers(1, 25))
        dtype = [np.int64, np.float64][trial % 2]
        w = rand_vector(rng, n, int(rng.integers(0, n + 1)), dtype, 0, 9, dense=bool(rng.random() < 0.6))
        mode = ["none", "normal", "complement"][int(rng.integers(0, 3))]
        mask = None if mode == "none" else rand_mask(rng, n, bool(rng.random() < 0.5))
        desc = make_desc(mode)
        kind = trial % 4
        w0 = vec_json(w)
        try:
            if kind == 0:
                val = 7
                idxs = None if rng.random() < 0.5 else sorted(rng.choice(n, size=int(rng.integers(0, n + 1)), replace=False).tolist())
                out = ref.assign(w, val, mask=mask, desc=desc, indices=idxs)
                extra = dict(value=val, indices=idxs)
            elif kind == 1:
                vals = rand_vector(rng, n, int(rng.integers(0, n + 1)), dtype, 0, 50, dense=bool(rng.random() < 0.5))
                tg = rand_vector(rng, n, int(rng.integers(0, n + 1)), np.int64, 0, n - 1, dense=bool(rng.random() < 0.5))
                out = ref.assign_scatter(w, vals, tg, mask=mask, desc=desc)
                extra = dict(values=vec_json(vals), targets=vec_json(tg))
            elif kind == 2:
                src = rand_vector(rng, n, int(rng.integers(0, n + 1)), dtype, 0, 50, dense=bool(rng.random() < 0.5))
                ix = rand_vector(rng, n, int(rng.integers(0, n + 1)), np.int64, 0, n - 1, dense=bool(rng.random() < 0.5))
                out = ref.extract_gather(w, src, ix, mask=mask, desc=desc)
                extra = dict(src=vec_json(src), idx=vec_json(ix))
            else:
                out = ref.apply(lambda x: x * 3 + 1, w, mask=mask, desc=desc)
                extra = dict(fn="affine", scale=3, shift=1)
            err = None
        except Exception as exc:
            out, err = None, type(exc).__name__
        add("assign", variant=["assign", "scatter", "gather", "apply"][kind], w=w0,
            mask=vec_json(mask), mask_mode=mode, out=vec_json(out), error=err, **extra)

    for trial in range(24):
        n = int(rng.integers(1, 30))
        dtype = [np.int64, np.float64][trial % 2]
        u = rand_vector(rng, n, int(rng.integers(0, n + 1)), dtype, -4, 9, dense=bool(trial % 3 == 0))
        mname = ["Plus", "Multiplies", "Minimum", "Maximum", "LogicalOr", "LogicalAnd"][trial % 6]
        r = ref.reduce(ref.builtin_monoid(mname), u)
        A = rand_matrix(rng, n, n, 0.3, dtype, -4, 9)
        rr = ref.reduce_rows(ref.builtin_monoid(mname), A)
        rs = ref.reduce_scalar_matrix(ref.builtin_monoid(mname), A)
        add("reduce", monoid=mname, u=vec_json(u), out=np.asarray(r).item(), A=mat_json(A),
            rows=vec_json(rr), scalar=np.asarray(rs).item())
    return cases


# ---------------------------------------------------------------------------
# round-2 pins: weights, non-integral SSSP and per-iteration PageRank at the
# BASELINE scales, the uniform family at s16 (written to pins.json)
# ---------------------------------------------------------------------------

PIN_SAMPLES = 256


def sample_ids(n, seed=7):
    """Vertex 0 (the R-MAT hub) plus PIN_SAMPLES-1 seeded vertex ids."""
    rng = np.random.default_rng(seed)
    return np.unique(np.concatenate([[0], rng.integers(0, n, PIN_SAMPLES - 1)])).astype(np.int64)


def pr_replay(A, alpha=0.85, iters=20):
    """algorithms.py:153-161 replayed with the reference's own kernels, one
    record per iteration (the reference's pagerank(max_iters=k) returns the
    k-th of these)."""
    from graphalg.algorithms import _scale_rows
    from graphalg.algebra import MINUS, TIMES
    pt = ref.builtin_semiring("PlusMultiplies")
    plus = ref.builtin_monoid("Plus")
    n = A.nrows
    scaled = _scale_rows(A, alpha)
    teleport = (1.0 - alpha) / n
    ranks = ref.Vector.filled(n, 1.0 / n)
    ids = sample_ids(n)
    out = []
    for _ in range(iters):
        previous = ranks
        spread = ref.vxm(pt, previous, scaled, desc=ref.Descriptor())
        ranks = ref.ewise_add(pt, spread, teleport, desc=ref.Descriptor())
        delta = ref.ewise_mult(MINUS, ranks, previous, desc=ref.Descriptor())
        squared = ref.ewise_add(TIMES, delta, delta, desc=ref.Descriptor())
        err = float(np.sqrt(float(ref.reduce(plus, squared))))
        v = np.asarray(ranks.values, dtype=np.float64)
        out.append(dict(sum=float(v.sum()), sumsq=float(np.dot(v, v)), error=err,
                        digest9=ref_cli._digest(ranks), samples=[float(x) for x in v[ids]]))
    final = ref.pagerank(A, alpha=alpha, eps=1e-300, max_iters=iters)
    assert np.array_equal(np.asarray(final.values), v), "replay differs from pagerank()"
    return dict(sample_ids=ids.tolist(), iterations=out)


def make_pins(scales_w=(16, 18, 20), scales_pr=(16, 20)):
    res = dict(note="reference outputs (graphalg 0.1.0, /root/reference/pkg) computed in the "
                    "build container by tests/golden/make_golden.py --only pins")
    for s in scales_w:
        t = time.time()
        W = build(s, weighted=True)
        res[f"weights_rmat_s{s}"] = dict(digest=values_digest(W.csr_values), nnz=int(W.nnz),
                                         sum=float(W.csr_values.sum()))
        if s in (16, 20):
            # the non-integral variant of C2: sqrt of the reference weights,
            # fed as the same CSR to both sides
            Wn = ref.SparseMatrix.from_csr(W.nrows, W.ncols, W.row_offsets.copy(),
                                           W.col_indices.copy(), np.sqrt(W.csr_values))
            desc = ref.Descriptor()
            dist = ref.sssp(Wn, 0, desc=desc)
            v = np.asarray(dist.values)
            ids = sample_ids(W.nrows)
            fin = np.isfinite(v)
            res[f"sssp_sqrt_s{s}"] = dict(digest=ref_cli._digest(dist), trace=trace_of(desc),
                                          finite=int(fin.sum()), sum_finite=float(v[fin].sum()),
                                          sample_ids=ids.tolist(),
                                          samples=[float(x) if np.isfinite(x) else None for x in v[ids]])
        del W
        print(f"pins weights s{s} {time.time()-t:.1f}s", flush=True)
    for s in scales_pr:
        t = time.time()
        res[f"pr_iter_s{s}"] = pr_replay(build(s))
        print(f"pins pr s{s} {time.time()-t:.1f}s", flush=True)
    uni = dict(a=0.25, b=0.25, c=0.25, d=0.25)
    for s in (14, 16):
        t = time.time()
        A = build(s, **uni)
        W = build(s, weighted=True, **uni)
        desc = ref.Descriptor()
        lv = ref.bfs(A, 0, desc=desc)
        dd = ref.Descriptor()
        cc = ref.connected_components(A, desc=dd)
        res[f"uniform_s{s}"] = dict(nnz=int(A.nnz), csr=csr_digest(A),
                                    weights=values_digest(W.csr_values),
                                    bfs=dict(digest=ref_cli._digest(lv), trace=trace_of(desc)),
                                    cc=dict(digest=ref_cli._digest(cc), trace=trace_of(dd)),
                                    sssp=dict(digest=ref_cli._digest(ref.sssp(W, 0))),
                                    tc=int(ref.triangle_count(A)))
        print(f"pins uniform s{s} {time.time()-t:.1f}s", flush=True)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--only", default="all")
    args = ap.parse_args()
    if args.only in ("all", "kernels"):
        cases = kernel_cases()
        with open(os.path.join(HERE, "kernel_cases.json"), "w") as fh:
            json.dump(cases, fh, separators=(",", ":"))
        print(f"kernel cases: {len(cases)}", flush=True)
    if args.only in ("all", "graphs"):
        out = {}
        make_graphs(out, [8, 10, 12, 14, 16] + ([18, 20] if args.big else []))
        with open(os.path.join(HERE, "rmat_graphs.json"), "w") as fh:
            json.dump(out, fh, indent=1)
    if args.only == "pins":
        res = make_pins()
        with open(os.path.join(HERE, "pins.json"), "w") as fh:
            json.dump(res, fh, indent=1)
        return
    if args.only in ("all", "algorithms"):
        res = run_algorithms([8, 10, 12, 14, 16] + ([18, 20] if args.big else []),
                             [8, 10, 12, 14] + ([16, 20] if args.big else []), args.big)
        with open(os.path.join(HERE, "algorithms.json" if not args.big else "algorithms_big.json"), "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
