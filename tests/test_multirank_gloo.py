"""World-size-2 `gloo` tests of the multi-GPU row partition, on CPU.

The GPU path exchanges X's row blocks and the canonical trace-block partials with
NCCL inside libellpack; the pool has one GPU, so here the same protocol runs over
gloo with the CPU oracle as the per-rank compute: each rank computes only its
256-aligned row block, the blocks and partials are all-gathered, and the
assembled result must be bitwise the single-process result (c12). The
bootstrap helpers bench.py uses (unique-id broadcast, max over ranks) run here
unchanged.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as tmp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _x2_rows(X, r0, r1, width, tau):
    """Oracle X^2 of rows [r0, r1) only (the rank's share): rows outside the block are empty in A."""
    import oracle
    from synth import Ell
    A = Ell.empty(X.n, X.w)
    A.val[r0:r1], A.col[r0:r1], A.nnz[r0:r1] = X.val[r0:r1], X.col[r0:r1], X.nnz[r0:r1]
    Y = Ell.empty(X.n, width)
    r = oracle.multiply(A, X, Y, 1.0, 0.0, tau, want_diag=True)
    return r, Y


def _worker(rank, ws, port, n, m, tau):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import oracle
    import synth
    from paper_2102_08505_b200 import multirank as mr

    oracle.set_threads(1)
    dist = mr.init_process_group("gloo")
    assert mr.dist_env() == (ws, rank, rank)

    # (1) NCCL unique-id bootstrap: rank 0's 128 bytes reach every rank unchanged
    uid = mr.broadcast_bytes(os.urandom(128) if rank == 0 else None)
    seen = [None] * ws
    dist.all_gather_object(seen, uid)
    assert len(uid) == 128 and all(s == uid for s in seen)

    # (2) the rank's 256-aligned block
    r0, r1 = mr.rank_rows(n, ws, rank)
    assert r0 % 256 == 0 and (r1 - r0) == n // ws

    X = synth.cfg5(n, m)
    ref_lit = oracle.x2(X, synth.Ell.empty(n, m), tau)  # literal width -> OVERFLOW report (R2)
    assert ref_lit.status == oracle.OVERFLOW
    w = ((ref_lit.required_width + 31) // 32) * 32
    ref_Y = synth.Ell.empty(n, w)
    ref = oracle.x2(X, ref_Y, tau)
    assert ref.status == oracle.OK

    # (3) overflow decision: per-rank counts all-reduced (sum rows, max width) = the P = 1 report
    r_lit, _ = _x2_rows(X, r0, r1, m, tau)
    assert r_lit.status == oracle.OVERFLOW
    assert int(mr.sum_over_ranks(r_lit.overflow_rows)) == ref_lit.overflow_rows
    assert int(mr.max_over_ranks(r_lit.required_width)) == ref_lit.required_width

    # (4) the rank's rows at the agreed width, then the all-gather of row blocks
    r, Y = _x2_rows(X, r0, r1, w, tau)
    assert r.status == oracle.OK
    blocks = {}
    for name in ("val", "col", "nnz"):
        mine = torch.from_numpy(np.ascontiguousarray(getattr(Y, name)[r0:r1]))
        parts = [torch.empty_like(mine) for _ in range(ws)]
        dist.all_gather(parts, mine)
        blocks[name] = torch.cat(parts).numpy()
    assert np.array_equal(blocks["nnz"], ref_Y.nnz)
    for i in range(n):
        k = int(ref_Y.nnz[i])
        assert np.array_equal(blocks["col"][i, :k], ref_Y.col[i, :k])
        assert np.array_equal(blocks["val"][i, :k].view(np.uint64), ref_Y.val[i, :k].view(np.uint64))

    # (5) canonical traces: own block partials all-gathered (never all-reduced), summed in block order
    diag_x = np.zeros(n)
    for i in range(r0, r1):
        hit = X.col[i, :X.nnz[i]] == i
        diag_x[i] = X.val[i, :X.nnz[i]][hit][0] if hit.any() else 0.0
    for d, expect in ((diag_x, ref.trace_x), (r.diag_s, ref.trace_x2)):
        own = torch.from_numpy(oracle.block_partials(d)[r0 // 256:r1 // 256].copy())
        parts = [torch.empty_like(own) for _ in range(ws)]
        dist.all_gather(parts, own)
        total = 0.0
        for t in torch.cat(parts).tolist():
            total = total + t
        assert np.float64(total).view(np.uint64) == np.float64(expect).view(np.uint64)

    # (6) bench.py timing: the slowest rank decides
    assert mr.max_over_ranks(1.5 + rank) == 1.5 + (ws - 1)
    dist.barrier()
    dist.destroy_process_group()


def _halo_worker(rank, ws, port, n, m, tau):
    """§8f-f1: each rank holds only its own block of X; the library's halo plan
    (ellpack_halo_plan, the function ellpack_halo_rows runs) moves exactly the rows its own rows
    reference; the rank's X^2 rows computed from that partial X are bitwise the full result."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import oracle
    import synth
    import paper_2102_08505_b200 as eb
    from paper_2102_08505_b200 import multirank as mr

    oracle.set_threads(1)
    dist = mr.init_process_group("gloo")
    r0, r1 = mr.rank_rows(n, ws, rank)
    per = r1 - r0
    X = synth.cfg5(n, m)
    # this rank's view: own block only
    Xr = synth.Ell.empty(n, X.w)
    Xr.val[r0:r1], Xr.col[r0:r1], Xr.nnz[r0:r1] = X.val[r0:r1], X.col[r0:r1], X.nnz[r0:r1]
    own = [i for i in range(r0, r1) if X.nnz[i] > 0]
    need = (min(int(X.col[i, 0]) for i in own), max(int(X.col[i, X.nnz[i] - 1]) for i in own))
    needs = [None] * ws
    dist.all_gather_object(needs, need)
    sends, recvs = eb.halo_plan(n, ws, rank, per, needs)
    # every referenced row is either own or received, and nothing else is received
    got = set(range(r0, r1))
    for _, t0, t1 in recvs:
        got |= set(range(t0, t1))
    assert set(range(need[0], need[1] + 1)) <= got
    assert all(need[0] <= t0 and t1 <= need[1] + 1 for _, t0, t1 in recvs)
    # the sends of every rank are the receives of their peers (plans agree pairwise)
    all_s, all_r = [None] * ws, [None] * ws
    dist.all_gather_object(all_s, sends)
    dist.all_gather_object(all_r, recvs)
    for p_ in range(ws):
        for q, s0, s1 in all_s[p_]:
            assert (p_, s0, s1) in all_r[q]
    reqs = []
    for q, s0, s1 in sends:
        for name in ("val", "col", "nnz"):
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(getattr(Xr, name)[s0:s1])), q))
    bufs = []
    for q, t0, t1 in recvs:
        for name in ("val", "col", "nnz"):
            b = torch.from_numpy(np.ascontiguousarray(getattr(Xr, name)[t0:t1]).copy())
            bufs.append((name, t0, t1, b))
            reqs.append(dist.irecv(b, q))
    for r in reqs:
        r.wait()
    for name, t0, t1, b in bufs:
        getattr(Xr, name)[t0:t1] = b.numpy()
    # own rows of X^2 from the partial view == the full computation
    A = synth.Ell.empty(n, X.w)
    A.val[r0:r1], A.col[r0:r1], A.nnz[r0:r1] = X.val[r0:r1], X.col[r0:r1], X.nnz[r0:r1]
    full = synth.Ell.empty(n, n)
    part = synth.Ell.empty(n, n)
    oracle.multiply(A, X, full, 1.0, 0.0, tau)
    oracle.multiply(A, Xr, part, 1.0, 0.0, tau)
    assert np.array_equal(part.nnz[r0:r1], full.nnz[r0:r1])
    for i in range(r0, r1):
        k = int(full.nnz[i])
        assert np.array_equal(part.col[i, :k], full.col[i, :k])
        assert np.array_equal(part.val[i, :k].view(np.uint64), full.val[i, :k].view(np.uint64))
    # the halo moved less than the all-gather would have
    moved = sum(t1 - t0 for _, t0, t1 in recvs)
    assert moved <= n - per
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("ws,n,m", [(2, 2048, 32), (4, 4096, 16), (4, 2048, 64)])
def test_halo_exchange_plan_gloo(ws, n, m):
    tmp.spawn(_halo_worker, args=(ws, _free_port(), n, m, 1e-5), nprocs=ws, join=True)


def _split_worker(rank, ws, port, n, m, tau):
    """§8f-f1 overlap: the interior rows of a rank's block (ellpack_row_split with the all-reduced
    half-bandwidth) reference only the rank's own rows, so they are computed BEFORE the halo arrives
    from the own block alone; the boundary rows, computed after it, reference only own + received
    rows; both phases reproduce the full result bit for bit and together cover the block."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import oracle
    import synth
    import paper_2102_08505_b200 as eb
    from paper_2102_08505_b200 import multirank as mr

    oracle.set_threads(1)
    dist = mr.init_process_group("gloo")
    r0, r1 = mr.rank_rows(n, ws, rank)
    X = synth.cfg5(n, m)
    rows = [i for i in range(r0, r1) if X.nnz[i] > 0]
    h_mine = max(max(i - int(X.col[i, 0]), int(X.col[i, X.nnz[i] - 1]) - i) for i in rows)
    h = int(mr.max_over_ranks(h_mine))
    (i0, i1), (l0, l1), (u0, u1) = eb.row_split(r0, r1, h)
    assert l0 == r0 and l1 == i0 and u0 == i1 and u1 == r1 and i0 <= i1
    own = synth.Ell.empty(n, X.w)
    own.val[r0:r1], own.col[r0:r1], own.nnz[r0:r1] = X.val[r0:r1], X.col[r0:r1], X.nnz[r0:r1]
    for i in range(i0, i1):  # interior: every referenced row is the rank's own
        k = int(X.nnz[i])
        assert k == 0 or (r0 <= X.col[i, 0] and X.col[i, k - 1] < r1)
    need = (min(int(X.col[i, 0]) for i in rows), max(int(X.col[i, X.nnz[i] - 1]) for i in rows))
    needs = [None] * ws
    dist.all_gather_object(needs, need)
    _, recvs = eb.halo_plan(n, ws, rank, r1 - r0, needs)
    have = set(range(r0, r1))
    for _, t0, t1 in recvs:
        have |= set(range(t0, t1))
    halo = own.copy()
    for _, t0, t1 in recvs:  # what the exchange delivers
        halo.val[t0:t1], halo.col[t0:t1], halo.nnz[t0:t1] = X.val[t0:t1], X.col[t0:t1], X.nnz[t0:t1]

    def rows_of_product(B, a, b):
        A = synth.Ell.empty(n, X.w)
        A.val[a:b], A.col[a:b], A.nnz[a:b] = X.val[a:b], X.col[a:b], X.nnz[a:b]
        out = synth.Ell.empty(n, n)
        oracle.multiply(A, B, out, 1.0, 0.0, tau)
        return out

    full = rows_of_product(X, r0, r1)
    phase1 = rows_of_product(own, i0, i1)          # before the halo: own rows only
    for a, b in ((l0, l1), (u0, u1)):
        for i in range(a, b):                      # boundary rows: own + received suffice
            k = int(X.nnz[i])
            assert all(int(j) in have for j in X.col[i, :k])
    phase2 = rows_of_product(halo, r0, r1)         # after it (boundary rows; interior too)
    for i in range(r0, r1):
        got = phase1 if i0 <= i < i1 else phase2
        k = int(full.nnz[i])
        assert got.nnz[i] == k
        assert np.array_equal(got.col[i, :k], full.col[i, :k])
        assert np.array_equal(got.val[i, :k].view(np.uint64), full.val[i, :k].view(np.uint64))
    dist.barrier()
    dist.destroy_process_group()


def _sym_halo_worker(rank, ws, port, n, m, tau):
    """The symmetric SP2 step across ranks (§8f-f4 ii with a communicator): each rank computes the
    upper triangle U of its own rows of Y = drop(X^2); the rows it mirrors (U rows of lower ranks) come
    from the halo plan with need ranges [r0_q - 2 h_X, r1_q) -- X^2's band is at most twice X's --
    and every row assembled as L_i || U_i from own + received U rows is the full row, bit for bit."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import oracle
    import synth
    import paper_2102_08505_b200 as eb
    from paper_2102_08505_b200 import multirank as mr

    oracle.set_threads(1)
    dist = mr.init_process_group("gloo")
    r0, r1 = mr.rank_rows(n, ws, rank)
    per = r1 - r0
    X = synth.cfg5(n, m)  # bitwise symmetric
    rows = [i for i in range(r0, r1) if X.nnz[i] > 0]
    h = int(mr.max_over_ranks(max(max(i - int(X.col[i, 0]), int(X.col[i, X.nnz[i] - 1]) - i) for i in rows)))
    full = synth.Ell.empty(n, n)
    oracle.x2(X, full, tau)  # every row (reference)
    U = {}  # this rank's upper rows: (cols >= i, values)
    for i in range(r0, r1):
        k = int(full.nnz[i])
        c, v = full.col[i, :k], full.val[i, :k]
        U[i] = (c[c >= i].copy(), v[c >= i].copy())
    need = [(max(0, q * per - 2 * h), (q + 1) * per - 1) for q in range(ws)]
    sends, recvs = eb.halo_plan(n, ws, rank, per, need)
    assert all(p_ < rank for p_, _, _ in recvs) and all(p_ > rank for p_, _, _ in sends)  # one-sided
    got = {}
    # exchange as objects (host test of the plan; the library moves the rows by NCCL send/recv)
    box = [None] * ws
    dist.all_gather_object(box, {"sends": sends, "U": {j: (U[j][0].tolist(), U[j][1].tolist())
                                                     for q, s0, s1 in sends for j in range(s0, s1)}})
    for p_ in range(ws):
        for q, s0, s1 in box[p_]["sends"]:
            if q == rank:
                for j in range(s0, s1):
                    c, v = box[p_]["U"][j]
                    got[j] = (np.array(c, np.int32), np.array(v))
    avail = dict(got)
    avail.update(U)
    for i in range(r0, r1):  # assemble L_i || U_i
        L = [(j, avail[j][1][np.searchsorted(avail[j][0], i)]) for j in range(max(0, i - 2 * h), i)
             if j in avail and np.searchsorted(avail[j][0], i) < len(avail[j][0])
             and avail[j][0][np.searchsorted(avail[j][0], i)] == i]
        cols = [j for j, _ in L] + U[i][0].tolist()
        vals = np.array([v for _, v in L] + U[i][1].tolist())
        k = int(full.nnz[i])
        assert cols == full.col[i, :k].tolist(), i
        assert np.array_equal(vals.view(np.uint64), full.val[i, :k].view(np.uint64)), i
        # every row j whose U holds column i is available (own or received)
        assert all(j in avail for j in range(max(0, i - 2 * h), i) if i in set(full.col[j, :full.nnz[j]].tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("ws,n,m", [(2, 2048, 32), (4, 4096, 16)])
def test_symmetric_step_u_halo_gloo(ws, n, m):
    tmp.spawn(_sym_halo_worker, args=(ws, _free_port(), n, m, 1e-5), nprocs=ws, join=True)


@pytest.mark.parametrize("ws,n,m", [(2, 4096, 32), (4, 4096, 16)])
def test_interior_boundary_row_split_gloo(ws, n, m):
    tmp.spawn(_split_worker, args=(ws, _free_port(), n, m, 1e-5), nprocs=ws, join=True)


def test_halo_plan_rejects_bad_arguments():
    sys.path.insert(0, ROOT)
    import paper_2102_08505_b200 as eb
    with pytest.raises(eb.EllpackError):
        eb.halo_plan(1024, 2, 2, 512, [(0, 1), (0, 1)])  # rank out of range
    s, r = eb.halo_plan(1024, 2, 0, 512, [(0, 100), (900, 1023)])  # disjoint ranges: nothing moves
    assert s == [] and r == []


@pytest.mark.parametrize("n,m", [(2048, 64), (4096, 32)])
def test_row_partition_protocol_gloo_ws2(n, m):
    tmp.spawn(_worker, args=(2, _free_port(), n, m, 1e-5), nprocs=2, join=True)


def test_partition_rejects_unaligned_blocks():
    sys.path.insert(0, ROOT)
    from paper_2102_08505_b200 import multirank as mr
    assert mr.rank_rows(4096, 2, 1) == (2048, 4096)
    with pytest.raises(ValueError):
        mr.rank_rows(512 + 256, 2, 0)
