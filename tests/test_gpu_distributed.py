"""The 1D-partitioned BFS steps on one GPU: P ranks simulated in lock step,
and two real processes sharing the GPU over gloo.

Lock step: each simulated rank owns a BlockGraph and NativeSteps (its own
device buffers); the exchange runs FrontierExchange's protocol with the
collectives emulated by concatenating the ranks' tensors in rank order
(what allgather returns): counts, then the dense word slices
(gb_bfs_dist_pack_words / unpack_words) or the sparse id lists
(gb_bfs_dist_owned / set_ids).  Levels and the direction trace must equal
the single-GPU fused BFS for P = 1, 2, 3, 4, 8.
"""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def lockstep_exchange(ranks, g):
    """FrontierExchange with the allgathers emulated (rank-order concatenation)."""
    from paper_1908_01407_b200.distributed import FrontierExchange
    counts = torch.cat([st.owned().clone() for st in ranks])
    total = int(counts.sum())
    if total * 32 > g.n:
        wb, wmax = FrontierExchange().word_bounds(g, counts.device)
        gathered = torch.cat([st.pack_words(wmax).clone() for st in ranks])
        for st in ranks:
            st.unpack_words(gathered, wmax, wb)
    else:
        kmax = int(counts.max())
        gathered = torch.cat([st.owned_ids(kmax).clone() for st in ranks])
        for st in ranks:
            st.set_ids(gathered, counts, kmax)
    return total


def lockstep_bfs(A, P, source, desc, modes=None):
    from paper_1908_01407_b200.distributed import BlockGraph, NativeSteps, partition_bounds
    from paper_1908_01407_b200.kernels import DirectionDecision, direction_rule
    bounds = partition_bounds(A._csr.offsets.cpu().numpy(), P)
    ranks = [NativeSteps(BlockGraph.from_matrix(A, r, P, bounds)) for r in range(P)]
    g = ranks[0].g
    for st in ranks:
        st.init(source)
    modes = modes if modes is not None else set()
    K, depth = 1, 1
    iters = min(desc.max_niter, g.n + 1)
    for it in range(iters):
        chosen, est, thr = direction_rule(g.nnz, g.n, K, desc.switch_ratio, desc.direction)
        desc.direction_log.append(DirectionDecision(chosen, K, est, g.nnz, thr))
        for st in ranks:
            if chosen == "pull":
                st.pull(depth + 1)
            else:
                st.push(K)
        K = lockstep_exchange(ranks, g)
        modes.add("dense" if K * 32 > g.n else "sparse")
        Ks = [st.apply(depth + 1) for st in ranks]   # read back: must equal the exchanged K
        assert set(Ks) == {K}
        if K == 0:
            break
        depth += 1
        if it + 1 == iters:
            for st in ranks:
                st.unstamp(K)
    out = [st.levels.cpu().numpy() for st in ranks]
    for o in out[1:]:
        assert np.array_equal(o, out[0])
    return out[0]


@pytest.mark.parametrize("scale", [12, 16, 20])
@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_partitioned_equals_single(scale, P):
    import paper_1908_01407_b200 as gb
    A = gb.io.rmat_matrix(scale)
    for src in (0, 7):
        d1, d2 = gb.Descriptor(), gb.Descriptor()
        want = gb.bfs(A, src, desc=d1).values
        modes = set()
        got = lockstep_bfs(A, P, src, d2, modes)
        if P > 1 and src == 0:
            assert modes == {"dense", "sparse"}
        assert np.array_equal(got, want)
        assert [(x.chosen, x.frontier_nvals) for x in d1.direction_log] == \
            [(x.chosen, x.frontier_nvals) for x in d2.direction_log]


def lockstep_bfs_device(A, P, source, desc, extra=1, cut=False):
    """bfs_partitioned_device's protocol for P simulated ranks: every level
    the device-resident step, the dense word exchange (rank-order
    concatenation), the device-resident apply; `extra` no-op levels past the
    end, as the product loop enqueues them."""
    from paper_1908_01407_b200 import _lib
    from paper_1908_01407_b200.distributed import (BlockGraph, FrontierExchange, NativeSteps,
                                                   partition_bounds)
    from paper_1908_01407_b200.kernels import DirectionDecision
    bounds = partition_bounds(A._csr.offsets.cpu().numpy(), P)
    ranks = [NativeSteps(BlockGraph.from_matrix(A, r, P, bounds)) for r in range(P)]
    for st in ranks:
        st.prefix_cut = cut
    g = ranks[0].g
    iters = min(desc.max_niter, g.n + 1)
    policy = {"auto": _lib.DIR_AUTO, "force-push": _lib.DIR_PUSH,
              "force-pull": _lib.DIR_PULL}[desc.direction.value]
    for st in ranks:
        st.dev_init(source, iters, desc.switch_ratio, policy)
    wb, wmax = FrontierExchange().word_bounds(g, ranks[0].levels.device)
    left = None
    for it in range(iters):
        for st in ranks:
            st.dev_level()
        gathered = torch.cat([st.pack_words(wmax).clone() for st in ranks])
        for st in ranks:
            st.unpack_words(gathered, wmax, wb)
            st.dev_apply()
        done = {int(st.state[NativeSteps.STATE_DONE]) for st in ranks}
        assert len(done) == 1
        if left is None and done == {1}:
            left = extra
        if left is not None:
            if left == 0:
                break
            left -= 1
    states = [st.state.cpu().numpy() for st in ranks]
    logs = [st.log.cpu().numpy() for st in ranks]
    for a, b in zip(states[1:], logs[1:]):
        assert np.array_equal(a, states[0]) and np.array_equal(b, logs[0])
    n_it = int(states[0][NativeSteps.STATE_ITERS])
    raw = logs[0]
    for i in range(n_it):
        desc.direction_log.append(DirectionDecision(
            "pull" if raw[1 + 3 * i] == _lib.DIR_PULL else "push", int(raw[2 + 3 * i]),
            int(raw[3 + 3 * i]), g.nnz, g.nnz * desc.switch_ratio))
    out = [st.levels.cpu().numpy() for st in ranks]
    for o in out[1:]:
        assert np.array_equal(o, out[0])
    return out[0]


@pytest.mark.parametrize("scale", [12, 16, 20])
@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_device_resident_partitioned_equals_single(scale, P):
    """The device-resident level loop (direction rule, K, depth and exit on
    the device; dense exchange only): levels, decisions and estimates equal
    the single-GPU fused BFS, with no-op levels past the end."""
    import paper_1908_01407_b200 as gb
    A = gb.io.rmat_matrix(scale)
    for src, extra, cut in ((0, 1, False), (7, 3, False), (0, 1, True), (7, 2, True)):
        if True:
            d1, d2 = gb.Descriptor(), gb.Descriptor()
            want = gb.bfs(A, src, desc=d1).values
            got = lockstep_bfs_device(A, P, src, d2, extra, cut)
            assert np.array_equal(got, want)
            assert [(x.chosen, x.frontier_nvals, x.estimated_frontier_edges)
                    for x in d1.direction_log] == \
                [(x.chosen, x.frontier_nvals, x.estimated_frontier_edges)
                 for x in d2.direction_log]


@pytest.mark.parametrize("cap", [0, 1, 2, 3])
@pytest.mark.parametrize("direction", ["auto", "force-push", "force-pull"])
def test_device_resident_partitioned_caps_and_policies(cap, direction):
    import paper_1908_01407_b200 as gb
    from paper_1908_01407_b200 import distributed
    A = gb.io.rmat_matrix(14)
    dir_ = gb.Direction(direction)
    for P in (1, 3):
        d1 = gb.Descriptor(max_niter=cap, direction=dir_)
        d2 = gb.Descriptor(max_niter=cap, direction=dir_)
        want = gb.bfs(A, 5, desc=d1).values
        if cap == 0:
            g = distributed.BlockGraph.from_matrix(A, 0, 1)
            got = distributed.bfs_partitioned_device(g, 5, d2).cpu().numpy()
        else:
            got = lockstep_bfs_device(A, P, 5, d2)
        assert np.array_equal(got, want)
        assert [(x.chosen, x.frontier_nvals) for x in d1.direction_log] == \
            [(x.chosen, x.frontier_nvals) for x in d2.direction_log]


@pytest.mark.parametrize("P", [1, 2, 4])
def test_device_resident_ordered_layout_prefix_cut(P):
    """The degree-ordered partition (rank 0 owns the hubs) with the push's
    prefix cut: levels by original id and the trace equal the single GPU's."""
    import paper_1908_01407_b200 as gb
    from paper_1908_01407_b200.containers import SparseMatrix
    A = gb.io.rmat_matrix(18)
    push_o, pull_o, rank = A.traversal()
    Ar = SparseMatrix._wrap(A.nrows, A.ncols, push_o, pull_o, A.dtype, A._sym)
    rank = rank.long().cpu().numpy()
    for src in (0, 5, 100000):
        d1, d2 = gb.Descriptor(), gb.Descriptor()
        want = gb.bfs(A, src, desc=d1).values
        got_r = lockstep_bfs_device(Ar, P, int(rank[src]), d2, cut=True)
        assert np.array_equal(got_r[rank], want)
        assert [(x.chosen, x.frontier_nvals) for x in d1.direction_log] == \
            [(x.chosen, x.frontier_nvals) for x in d2.direction_log]


def test_device_resident_entry_single_rank():
    """The product loop itself at world size 1 (the exchange is local)."""
    import paper_1908_01407_b200 as gb
    from paper_1908_01407_b200 import distributed
    A = gb.io.rmat_matrix(16)
    g = distributed.BlockGraph.from_matrix(A, 0, 1)
    for src in (0, 3, 60000):
        for look in (1, 2, 4):
            d1, d2 = gb.Descriptor(), gb.Descriptor()
            want = gb.bfs(A, src, desc=d1).values
            got = distributed.bfs_partitioned_device(g, src, d2, lookahead=look).cpu().numpy()
            assert np.array_equal(got, want)
            assert [(x.chosen, x.frontier_nvals) for x in d1.direction_log] == \
                [(x.chosen, x.frontier_nvals) for x in d2.direction_log]


def lockstep_cc(A, P, desc, sparsify=True):
    from paper_1908_01407_b200.distributed import BlockGraph, NativeCCSteps, partition_bounds
    from paper_1908_01407_b200.kernels import DirectionDecision, direction_rule
    bounds = partition_bounds(A._csr.offsets.cpu().numpy(), P)
    ranks = [NativeCCSteps(BlockGraph.from_matrix(A, r, P, bounds)) for r in range(P)]
    g = ranks[0].g
    for st in ranks:
        st.init()
    live = g.n
    for _ in range(desc.max_niter):
        chosen, est, thr = direction_rule(g.nnz, g.n, live, desc.switch_ratio, desc.direction)
        desc.direction_log.append(DirectionDecision(chosen, live, est, g.nnz, thr))
        for st in ranks:
            st.hook_and_propose(chosen == "pull")
        total = ranks[0].prop.clone()
        for st in ranks[1:]:
            total = torch.minimum(total, st.prop)
        for st in ranks:
            st.prop.copy_(total)
        outs = [st.shortcut(sparsify) for st in ranks]
        assert len(set(outs)) == 1
        changed, live = outs[0]
        if changed == 0:
            break
    res = [st.result().cpu().numpy() for st in ranks]
    for r in res[1:]:
        assert np.array_equal(r, res[0])
    return res[0]


@pytest.mark.parametrize("scale", [12, 18])
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_partitioned_cc_equals_single(scale, P):
    import paper_1908_01407_b200 as gb
    A = gb.io.rmat_matrix(scale)
    for sparsify in (True, False):
        d1, d2 = gb.Descriptor(), gb.Descriptor()
        want = gb.connected_components(A, desc=d1, sparsify=sparsify).values
        got = lockstep_cc(A, P, d2, sparsify)
        assert np.array_equal(got, want)
        assert [(x.chosen, x.frontier_nvals) for x in d1.direction_log] == \
            [(x.chosen, x.frontier_nvals) for x in d2.direction_log]


def test_partitioned_world1_entry_point():
    import paper_1908_01407_b200 as gb
    from paper_1908_01407_b200 import distributed
    A = gb.io.rmat_matrix(14)
    d = gb.Descriptor(max_niter=3)
    got = distributed.bfs(A, 0, desc=d).values
    want = gb.bfs(A, 0, desc=gb.Descriptor(max_niter=3)).values
    assert np.array_equal(got, want)


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_partitioned_ordered_layout_equals_single(P):
    """The partition of the degree-ordered layout (OrderedPartitionedBfs
    blocks) in lock step: levels by original id equal the single-GPU BFS."""
    import paper_1908_01407_b200 as gb
    from paper_1908_01407_b200.containers import SparseMatrix
    A = gb.io.rmat_matrix(16)
    push_o, pull_o, rank = A.traversal()
    Ar = SparseMatrix._wrap(A.nrows, A.ncols, push_o, pull_o, A.dtype, A._sym)
    rank = rank.long().cpu().numpy()
    for src in (0, 5, 40000):
        d1, d2 = gb.Descriptor(), gb.Descriptor()
        want = gb.bfs(A, src, desc=d1).values
        got_r = lockstep_bfs(Ar, P, int(rank[src]), d2)
        assert np.array_equal(got_r[rank], want)
        assert [(x.chosen, x.frontier_nvals) for x in d1.direction_log] == \
            [(x.chosen, x.frontier_nvals) for x in d2.direction_log]


def test_ordered_partitioned_runner_single_rank():
    import paper_1908_01407_b200 as gb
    from paper_1908_01407_b200.distributed import OrderedPartitionedBfs
    A = gb.io.rmat_matrix(14)
    run = OrderedPartitionedBfs(A, 0, 1)
    for src in (0, 3, 9999):
        assert np.array_equal(run(src).cpu().numpy(), gb.bfs(A, src).values)


# ---------------------------------------------------------------------------
# two processes, one GPU, gloo: the product loop with NativeSteps and the
# real FrontierExchange collectives (NCCL needs one GPU per rank)
# ---------------------------------------------------------------------------


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _gloo_worker(rank, world, port_, scale, results):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1908_01407_b200 as gb
    from paper_1908_01407_b200 import distributed as gbd
    A = gb.io.rmat_matrix(scale)
    out = {}
    for ordered in (False, True):
        d = gb.Descriptor()
        if ordered:
            run = gbd.OrderedPartitionedBfs(A, rank, world, loop="host")
            lv = run(0, d).cpu().numpy()
            log = run.exchange.log
        else:
            g = gbd.BlockGraph.from_matrix(A, rank, world)
            ex = gbd.FrontierExchange()
            lv = gbd.bfs_partitioned(g, 0, d, exchange=ex).cpu().numpy()
            log = ex.log
        out[ordered] = (lv, [(x.chosen, x.frontier_nvals) for x in d.direction_log], list(log))
    d = gb.Descriptor()
    g = gbd.BlockGraph.from_matrix(A, rank, world)
    ex = gbd.FrontierExchange()
    lv = gbd.bfs_partitioned_device(g, 0, d, exchange=ex).cpu().numpy()
    out["device"] = (lv, [(x.chosen, x.frontier_nvals) for x in d.direction_log], list(ex.log))
    d = gb.Descriptor()
    lv = gbd.OrderedPartitionedBfs(A, rank, world)(0, d).cpu().numpy()   # default: device loop
    out["device_ordered"] = (lv, [(x.chosen, x.frontier_nvals) for x in d.direction_log])
    d = gb.Descriptor()
    lab = gbd.connected_components(A, d).values
    out["cc"] = lab
    results[rank] = out
    dist.destroy_process_group()


@pytest.mark.parametrize("scale", [14, 18])
def test_two_processes_gloo_native_steps(scale):
    import torch.multiprocessing as mp
    import paper_1908_01407_b200 as gb
    ctx = mp.get_context("spawn")
    results = ctx.Manager().dict()
    port_ = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port_, scale, results)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    A = gb.io.rmat_matrix(scale)
    d = gb.Descriptor()
    want = gb.bfs(A, 0, desc=d).values
    trace = [(x.chosen, x.frontier_nvals) for x in d.direction_log]
    want_cc = gb.connected_components(A).values
    for r in range(2):
        for ordered in (False, True):
            lv, tr, log = results[r][ordered]
            assert np.array_equal(lv, want)
            assert tr == trace
            assert {m for m, _b in log} == {"dense", "sparse"}
        lv, tr, log = results[r]["device"]
        assert np.array_equal(lv, want) and tr == trace
        assert {m for m, _b in log} == {"dense"} and len(log) == len(trace) + 1
        lv, tr = results[r]["device_ordered"]
        assert np.array_equal(lv, want) and tr == trace
        assert np.array_equal(results[r]["cc"], want_cc)
