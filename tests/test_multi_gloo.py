"""World-size-2 (gloo, CPU) test of the multi-GPU decomposition.

The engine row-shards CSR(A) and CSR(A^T) with equil_partition_rows, keeps
e.*s and d.*w in a padded layout (rank g owns slots [g*max, g*max + cnt_g)),
and all-gathers the slices after every fused pass (engine.cu allgather_padded).
Each row's sum stays on one rank, so the trajectory must be bit-identical to
the single-process run for any world size.  This test runs that exact
decomposition on CPU: the partition comes from the product library, the
per-row arithmetic from the oracle (test infrastructure), the exchange from
torch.distributed (gloo).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def det_exp_np(x):
    """numpy restatement of eo_det_exp (elementwise IEEE ops, no FMA)."""
    x = np.clip(x, -708.39, 709.78)
    fx = np.floor(1.4426950408889634073599 * x + 0.5)
    r = x - fx * 6.93145751953125E-1
    r = r - fx * 1.42860682030941723212E-6
    rr = r * r
    px = (1.26177193074810590878E-4 * rr + 3.02994407707441961300E-2) * rr
    px = (px + 9.99999999999999999910E-1) * r
    qx = ((3.00198505138664455042E-6 * rr + 2.52448340349684104192E-3) * rr
          + 2.27265548208155028766E-1) * rr + 2.00000000000000000009E0
    y = 2.0 * (px / (qx - px)) + 1.0
    k = fx.astype(np.int64)
    k1 = (k / 2).astype(np.int64)  # C truncation toward zero
    k1 = np.where(k < 0, -((-k) // 2), k // 2)
    k2 = k - k1
    return (y * np.ldexp(1.0, k1)) * np.ldexp(1.0, k2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, A_arrays, T, seed, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    import paper_1602_06621_b200 as eq
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, n, rp, col, val = A_arrays
    O = oracle.c_oracle()
    A = oracle.CsrArrays(m, n, rp, col, val)
    AT = O.transpose(A)
    ab = eq.partition_rows(rp, world)
    tb = eq.partition_rows(AT.row_ptr, world)
    amax = int(np.max(np.diff(ab)))
    tmax = int(np.max(np.diff(tb)))

    def local(C, b):
        r0, r1 = b[rank], b[rank + 1]
        k0, k1 = C.row_ptr[r0], C.row_ptr[r1]
        return oracle.CsrArrays(r1 - r0, C.n, C.row_ptr[r0:r1 + 1] - k0, C.col[k0:k1],
                                C.val[k0:k1]), r0, r1

    Al, a0, a1 = local(A, ab)
    Tl, t0, t1 = local(AT, tb)
    alpha, beta = np.sqrt(np.sqrt(n / m)), np.sqrt(np.sqrt(m / n))  # auto targets
    alpha, beta = eq.resolve_targets(eq.EquilibrationParams(), m, n)
    gamma, M = 0.1, 9.210340371976184
    bits = O.sign_bits(seed, 17, 0, T * (n + m) + 64)

    def sgn(g):
        return np.where((bits[g >> 5] >> (g & 31)) & 1, 1.0, -1.0)

    def gather(loc, cnt, mx, bounds, full):
        pad = torch.zeros(mx * world, dtype=torch.float64)
        pad[rank * mx: rank * mx + cnt] = torch.from_numpy(loc)
        parts = [torch.zeros(mx, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, pad[rank * mx:(rank + 1) * mx])
        outv = np.zeros(full)
        for g in range(world):
            c = bounds[g + 1] - bounds[g]
            outv[bounds[g]:bounds[g + 1]] = parts[g].numpy()[:c]
        return outv

    u = np.zeros(a1 - a0); ub = np.zeros(a1 - a0)
    v = np.zeros(t1 - t0); vb = np.zeros(t1 - t0)
    xs = sgn(np.arange(n, dtype=np.int64))            # e = 1
    xw = sgn(n + np.arange(m, dtype=np.int64))        # d = 1

    def upd(x, avg, est, lin, t):
        step = 2.0 / (gamma * float(t + 1))
        aw = 2.0 / (float(t) + 2.0)
        g = (est - lin) + gamma * x
        xi = x - step * g
        xi = np.where(xi < -M, -M, xi)
        xi = np.where(M < xi, M, xi)
        return xi, aw * xi + (1.0 - aw) * avg

    for t in range(1, T + 1):
        y = O.apply(Al, xs) * np.abs(xw[a0:a1])
        z = O.apply(Tl, xw) * np.abs(xs[t0:t1])
        u, ub = upd(u, ub, y * y, alpha * alpha, t)
        v, vb = upd(v, vb, z * z, beta * beta, t)
        if t == T:
            break
        base = t * (n + m)
        xw_loc = det_exp_np(u) * sgn(base + n + np.arange(a0, a1, dtype=np.int64))
        xs_loc = det_exp_np(v) * sgn(base + np.arange(t0, t1, dtype=np.int64))
        xw = gather(xw_loc, a1 - a0, amax, ab, m)
        xs = gather(xs_loc, t1 - t0, tmax, tb, n)
    U = gather(ub, a1 - a0, amax, ab, m)
    V = gather(vb, t1 - t0, tmax, tb, n)
    if rank == 0:
        out_q.put((U, V, ab.tolist(), tb.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_trajectory_bit_identical_world2(golden):
    from conftest import csr_from_golden
    import oracle
    A = csr_from_golden(golden, "lr")  # long rows, empty rows/columns
    T, seed = 6, 4
    want = oracle.c_oracle().sgd_equilibrate(A, iterations=T, seed=seed)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, (A.m, A.n, A.row_ptr, A.col, A.val),
                                               T, seed, q)) for r in range(2)]
    for p in procs:
        p.start()
    U, V, ab, tb = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert 0 < ab[1] < A.m and 0 < tb[1] < A.n  # both ranks own rows
    assert np.array_equal(U, want.u)
    assert np.array_equal(V, want.v)


def test_det_exp_numpy_restatement_matches_oracle(C):
    x = np.random.default_rng(2).uniform(-30, 30, 5000)
    assert np.array_equal(det_exp_np(x), C.det_exp(x))


def _lsqr_worker(rank, world, port, A_arrays, b, iters, out_q):
    """Row-sharded LSQR exactly as engine.cu lsqr_core runs it for world > 1:
    local slices of u / r (rows of A) and v / w / x (rows of A^T), the gathered
    d.*u, e.*v, e.*x exchanged after every update, every norm the canonical
    reduction of the whole (gathered) vector."""
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    import paper_1602_06621_b200 as eq
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, n, rp, col, val = A_arrays
    O = oracle.c_oracle()
    A = oracle.CsrArrays(m, n, rp, col, val)
    AT = O.transpose(A)
    ab = eq.partition_rows(rp, world)
    tb = eq.partition_rows(AT.row_ptr, world)
    amax, tmax = int(np.max(np.diff(ab))), int(np.max(np.diff(tb)))

    def local(C, bd):
        r0, r1 = bd[rank], bd[rank + 1]
        k0, k1 = C.row_ptr[r0], C.row_ptr[r1]
        return oracle.CsrArrays(r1 - r0, C.n, C.row_ptr[r0:r1 + 1] - k0, C.col[k0:k1],
                                C.val[k0:k1]), r0, r1

    Al, a0, a1 = local(A, ab)
    Tl, t0, t1 = local(AT, tb)

    def gather(loc, mx, bounds, full):
        pad = torch.zeros(mx, dtype=torch.float64)
        pad[:loc.size] = torch.from_numpy(loc)
        parts = [torch.zeros(mx, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, pad)
        outv = np.zeros(full)
        for g in range(world):
            outv[bounds[g]:bounds[g + 1]] = parts[g].numpy()[:bounds[g + 1] - bounds[g]]
        return outv

    def gnorm(loc, mside):
        full = gather(loc, amax, ab, m) if mside else gather(loc, tmax, tb, n)
        return np.sqrt(O.canon_sumsq(full))

    bnorm = np.sqrt(O.canon_sumsq(b))
    bl = b[a0:a1]
    hist = [1.0]
    x = np.zeros(t1 - t0)
    beta = gnorm(bl, True)
    u = bl / beta
    v = O.apply(Tl, gather(u, amax, ab, m))
    alpha = gnorm(v, False)
    v = v / alpha
    w = v.copy()
    phibar, rhobar = beta, alpha
    for _ in range(iters):
        un = O.apply(Al, gather(v, tmax, tb, n)) - alpha * u
        beta = gnorm(un, True)
        u = un / beta
        vn = O.apply(Tl, gather(u, amax, ab, m)) - beta * v
        alpha = gnorm(vn, False)
        v = vn / alpha
        rho = float(np.hypot(rhobar, beta))
        cs, sn = rhobar / rho, beta / rho
        theta = sn * alpha
        rhobar = -cs * alpha
        phi = cs * phibar
        phibar = sn * phibar
        x = x + (phi / rho) * w
        w = v - (theta / rho) * w
        r = bl - O.apply(Al, gather(x, tmax, tb, n))
        hist.append(gnorm(r, True) / bnorm)
    X = gather(x, tmax, tb, n)
    if rank == 0:
        out_q.put((np.array(hist), X))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_lsqr_bit_identical_world2(golden):
    from conftest import csr_from_golden
    import oracle
    A = csr_from_golden(golden, "sp")
    b = golden["sp_b"]
    iters = 12
    want = oracle.c_oracle().lsqr(A, b, iters, 0.0)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_lsqr_worker,
                         args=(r, 2, port, (A.m, A.n, A.row_ptr, A.col, A.val), b, iters, q))
             for r in range(2)]
    for p in procs:
        p.start()
    hist, X = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(hist, want.residual_history)
    assert np.array_equal(X, want.x)


def _transpose_worker(rank, world, port, A_arrays, out_q):
    """The sharded setup of engine.cu create_sharded on CPU: local rows of A,
    local transpose, global A^T row pointers as the all-reduced sum of the local
    prefix sums, all-to-all of the A^T row ranges (counts, columns, values), and
    the rank-order merge."""
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    import paper_1602_06621_b200 as eq
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, n, rp, col, val = A_arrays
    O = oracle.c_oracle()
    ab = eq.partition_rows(rp, world)
    a0, a1 = ab[rank], ab[rank + 1]
    k0, k1 = rp[a0], rp[a1]
    Al = oracle.CsrArrays(a1 - a0, n, rp[a0:a1 + 1] - k0, col[k0:k1], val[k0:k1])
    Tl = O.transpose(Al)  # n x (a1 - a0), columns = local rows
    glob = torch.from_numpy(Tl.row_ptr.astype(np.int64).copy())
    dist.all_reduce(glob)  # sum of prefix sums = CSR(A^T)'s row pointers
    rpT = glob.numpy()
    tb = eq.partition_rows(rpT, world)
    cnt = np.diff(Tl.row_ptr)
    pieces = [(cnt[tb[h]:tb[h + 1]], Tl.col[Tl.row_ptr[tb[h]]:Tl.row_ptr[tb[h + 1]]] + a0,
               Tl.val[Tl.row_ptr[tb[h]]:Tl.row_ptr[tb[h + 1]]]) for h in range(world)]
    gathered = [None] * world
    dist.all_gather_object(gathered, pieces)  # all-to-all through a gather
    t0, t1 = tb[rank], tb[rank + 1]
    rows = []
    offs = [0] * world
    for j in range(t1 - t0):
        cs, vs = [], []
        for g in range(world):
            c, cc, vv = gathered[g][rank]
            o, k = offs[g], int(c[j])
            cs.append(cc[o:o + k])
            vs.append(vv[o:o + k])
            offs[g] += k
        rows.append((np.concatenate(cs), np.concatenate(vs)))
    out_q.put((rank, t0, t1, rpT, rows))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_setup_transpose_alltoall(golden, world):
    """Each rank's merged A^T shard equals the rows cut from the full
    transpose, bit for bit (explicit_matrix.cpp:117-125)."""
    from conftest import csr_from_golden
    import oracle
    A = csr_from_golden(golden, "sp")
    full = oracle.c_oracle().transpose(A)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_transpose_worker,
                         args=(r, world, port, (A.m, A.n, A.row_ptr, A.col, A.val), q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, t0, t1, rpT, rows in got:
        assert np.array_equal(rpT, full.row_ptr)
        for j, (c, v) in enumerate(rows):
            k0, k1 = full.row_ptr[t0 + j], full.row_ptr[t0 + j + 1]
            assert np.array_equal(c, full.col[k0:k1]) and np.array_equal(v, full.val[k0:k1])
