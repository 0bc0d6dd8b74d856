"""GPU checks of K3 (CGS2 step), K4 (combination) and the fp64 reductions.

Floating-point kernels: compared with an fp64 numpy reference of the same op
(MGS + reorthogonalisation, ctkrylov/arnoldi.py:66-82, for the Arnoldi step).
"""

import numpy as np
import pytest

from paper_2602_17892_b200.arnoldi import DeviceBasis

pytestmark = pytest.mark.gpu


def basis_with(torch, Q, rows):
    L, k1 = Q.shape
    B = DeviceBasis(L, rows, torch.device("cuda", 0), torch)
    B.W[:k1, :L] = torch.from_numpy(Q.T.astype(np.float32)).cuda()
    return B


@pytest.mark.parametrize("L,k", [(1000, 0), (4099, 5), (65536, 80), (130680, 30), (262147, 63),
                                 (1048576, 3), (2086560, 1), (4194309, 6),
                                 # streamed path: 256-float tiles (c4 / c5 sizes, last c4
                                 # step), 128-float tiles, ragged last tile and CTA ranges
                                 (2086560, 40), (2086560, 100), (4194304, 20), (1048576, 120),
                                 (600004, 9)])
def test_cgs2_step_matches_fp64_mgs(cuda, L, k):
    torch = cuda
    rng = np.random.default_rng(L + k)
    Q, _ = np.linalg.qr(rng.standard_normal((L, k + 1)))
    Q = Q.astype(np.float32).astype(np.float64)
    q = rng.standard_normal(L).astype(np.float32).astype(np.float64)
    B = basis_with(torch, Q, k + 3)
    qd = torch.from_numpy(q.astype(np.float32)).cuda()
    h = torch.zeros(k + 8, dtype=torch.float64, device="cuda")
    stat = torch.zeros(4, dtype=torch.float64, device="cuda")
    B.cgs2_step(k, qd, h, stat, torch.cuda.current_stream())
    torch.cuda.synchronize()
    # fp64 reference: MGS + one reorthogonalisation pass
    v = q.copy()
    href = np.zeros(k + 2)
    for _ in range(2):
        for i in range(k + 1):
            c = Q[:, i] @ v
            href[i] += c
            v = v - c * Q[:, i]
    href[k + 1] = np.linalg.norm(v)
    hg = h.cpu().numpy()[: k + 2]
    np.testing.assert_allclose(hg, href, rtol=1e-5, atol=1e-5 * np.abs(href).max())
    st = stat.cpu().numpy()
    assert st[0] == pytest.approx(np.linalg.norm(q), rel=1e-12)
    assert st[1] == 0.0
    w = B.W[k + 1, :L].cpu().numpy().astype(np.float64)
    np.testing.assert_allclose(w, v / href[k + 1], atol=2e-6)
    # new row is orthogonal to the basis to fp32 working precision
    assert np.abs(Q.T @ w).max() < 1e-5


def mgs2_ref(Q, q):
    """fp64 MGS + one reorthogonalisation pass (ctkrylov/arnoldi.py:66-82)."""
    v = q.copy()
    k1 = Q.shape[1]
    href = np.zeros(k1 + 1)
    for _ in range(2):
        for i in range(k1):
            c = Q[:, i] @ v
            href[i] += c
            v = v - c * Q[:, i]
    href[k1] = np.linalg.norm(v)
    return href, v


@pytest.mark.parametrize("L,K,near", [(32940, 50, False), (65536, 80, False),
                                      (65536, 30, True), (2086560, 40, False),
                                      (4194304, 24, False), (2086560, 12, True)])
def test_gram_corrected_cgs2_chain_matches_fp64_mgs(cuda, L, K, near):
    """Consecutive steps 0..K-1 on one basis take the Gram-corrected
    single-launch path (E = W^T W - I kept across steps; SMEM path for short
    vectors, streamed path for c4/c5 lengths).  Every step's column equals
    fp64 MGS + reorthogonalisation on the STORED fp32 rows, and the basis
    stays orthonormal to fp32 working precision.  near=True makes every q
    nearly dependent on the basis (||q2|| ~ 1e-6 ||q||): the norm estimate
    would cancel, so the kernels take the explicit-norm fallback."""
    torch = cuda
    rng = np.random.default_rng(L + K)
    B = DeviceBasis(L, K + 2, torch.device("cuda", 0), torch)
    v0 = rng.standard_normal(L)
    B.W[0, :L] = torch.from_numpy((v0 / np.linalg.norm(v0)).astype(np.float32)).cuda()
    st = torch.cuda.current_stream()
    h = torch.zeros(K + 8, dtype=torch.float64, device="cuda")
    stat = torch.zeros(4, dtype=torch.float64, device="cuda")
    worst = 0.0
    for k in range(K):
        Q = B.W[: k + 1, :L].cpu().numpy().astype(np.float64).T
        if near:
            p = Q @ rng.standard_normal(k + 1)
            u = rng.standard_normal(L)
            q = p + 1e-6 * np.linalg.norm(p) * u / np.linalg.norm(u)
        else:
            q = rng.standard_normal(L) + Q @ rng.standard_normal(k + 1)
        q = q.astype(np.float32).astype(np.float64)
        B.cgs2_step(k, torch.from_numpy(q.astype(np.float32)).cuda(), h, stat, st)
        torch.cuda.synchronize()
        href, v = mgs2_ref(Q, q)
        hg = h.cpu().numpy()[: k + 2]
        err = np.abs(hg - href).max() / np.abs(href).max()
        worst = max(worst, err)
        assert err < 1e-5, (k, err)
        assert hg[k + 1] == pytest.approx(href[k + 1], rel=1e-5), k
        w = B.W[k + 1, :L].cpu().numpy().astype(np.float64)
        assert np.abs(w - v / href[k + 1]).max() < 5e-6, k
    W = B.W[: K + 1, :L].cpu().numpy().astype(np.float64)
    G = W @ W.T
    assert np.abs(G - np.eye(K + 1)).max() < 2e-6, np.abs(G - np.eye(K + 1)).max()


def test_cgs2_breakdown_flag(cuda):
    torch = cuda
    L = 4096
    rng = np.random.default_rng(1)
    Q, _ = np.linalg.qr(rng.standard_normal((L, 3)))
    B = basis_with(torch, Q.astype(np.float32).astype(np.float64), 5)
    q = (Q[:, :3] @ np.array([1.0, -2.0, 0.5])).astype(np.float32)    # in span(W): invariant
    qd = torch.from_numpy(q).cuda()
    h = torch.zeros(8, dtype=torch.float64, device="cuda")
    stat = torch.zeros(4, dtype=torch.float64, device="cuda")
    # only rows 0..2 are basis rows: step k=2 orthogonalises against 3 rows
    B.cgs2_step(2, qd, h, stat, torch.cuda.current_stream())
    torch.cuda.synchronize()
    st = stat.cpu().numpy()
    # fp32 inputs leave a ~1e-7 relative residue: breakdown iff h <= 1e-14 ||q||
    assert st[3] <= 1e-5 * st[0]


@pytest.mark.parametrize("L,k", [(33, 4), (32940, 17), (130683, 77), (1000003, 40)])
def test_combine_and_norms(cuda, L, k):
    torch = cuda
    rng = np.random.default_rng(k)
    Wh = rng.standard_normal((k, L)).astype(np.float32)
    B = DeviceBasis(L, k + 1, torch.device("cuda", 0), torch)
    B.W[:k, :L] = torch.from_numpy(Wh).cuda()
    y = rng.standard_normal(k)
    x0 = rng.standard_normal(L).astype(np.float32)
    yd = torch.from_numpy(y).cuda()
    x0d = torch.from_numpy(x0).cuda()
    out = torch.empty(L, dtype=torch.float32, device="cuda")
    nrm = torch.zeros(1, dtype=torch.float64, device="cuda")
    B.combine(k, yd, out, x0=x0d, norm_out=nrm, stream=torch.cuda.current_stream())
    ref = x0.astype(np.float64) + Wh.astype(np.float64).T @ y
    got = out.cpu().numpy()
    np.testing.assert_allclose(got, ref, rtol=1e-6, atol=1e-5)
    assert nrm.item() == pytest.approx(float(np.sum(got.astype(np.float64) ** 2)), rel=1e-12)
    n2 = torch.zeros(1, dtype=torch.float64, device="cuda")
    B.norm2(x0d, n2, torch.cuda.current_stream())
    assert n2.item() == pytest.approx(float(np.sum(x0.astype(np.float64) ** 2)), rel=1e-12)
    dots = torch.zeros(k + 1, dtype=torch.float64, device="cuda")
    B.dots(k, x0d, dots, True, torch.cuda.current_stream())
    dref = Wh.astype(np.float64) @ x0.astype(np.float64)
    np.testing.assert_allclose(dots.cpu().numpy()[:k], dref, rtol=1e-10, atol=1e-9)


@pytest.mark.parametrize("Lx,Lr,k0,nb", [(4096, 32940, 1, 8), (65536, 130682, 41, 8),
                                         (1001, 2087, 75, 3), (16, 12, 5, 1)])
def test_iterate_batch_matches_per_iterate_combinations(cuda, Lx, Lr, k0, nb):
    """ctk_iterate_batch: one pass over X / AX for nb iterates gives the same
    norms and last iterate as the fp64 host combinations x0 + X y_b and
    d0 - AX y_b (fp32-rounded entries, fp64 sums)."""
    torch = cuda
    from paper_2602_17892_b200 import _native
    lib = _native.load()
    rng = np.random.default_rng(Lx + k0)
    rows = k0 + nb + 2
    ldx, ldr = (Lx + 3) // 4 * 4, (Lr + 3) // 4 * 4
    X = rng.standard_normal((rows, ldx)).astype(np.float32)
    AX = rng.standard_normal((rows, ldr)).astype(np.float32)
    x0 = rng.standard_normal(Lx).astype(np.float32)
    d0 = rng.standard_normal(Lr).astype(np.float32)
    Y = np.zeros((nb, rows))
    for b in range(nb):
        Y[b, :k0 + b] = rng.standard_normal(k0 + b)
    dev = torch.device("cuda", 0)
    Xd, AXd = torch.from_numpy(X).to(dev), torch.from_numpy(AX).to(dev)
    x0d, d0d = torch.from_numpy(x0).to(dev), torch.from_numpy(d0).to(dev)
    Yd = torch.from_numpy(Y).to(dev)
    x = torch.zeros(Lx, device=dev)
    r = torch.zeros(Lr, device=dev)
    norms = torch.zeros(2 * nb, dtype=torch.float64, device=dev)
    cap = rows + 2
    scratch = torch.zeros(int(lib.ctk_reduce_scratch_bytes(cap, Lr)) // 8 + 1,
                          dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream()
    for _ in range(2):          # the second call reuses the (reset) tickets
        _native.check(lib.ctk_iterate_batch(Xd.data_ptr(), ldx, x0d.data_ptr(), x.data_ptr(), Lx,
                                            AXd.data_ptr(), ldr, d0d.data_ptr(), r.data_ptr(), Lr,
                                            k0, nb, Yd.data_ptr(), rows, norms.data_ptr(),
                                            scratch.data_ptr(), cap, st.cuda_stream),
                      "ctk_iterate_batch")
    torch.cuda.synchronize()
    got = norms.cpu().numpy()
    for b in range(nb):
        k = k0 + b
        xr = x0.astype(np.float64) + X[:k, :Lx].astype(np.float64).T @ Y[b, :k]
        rr = d0.astype(np.float64) - AX[:k, :Lr].astype(np.float64).T @ Y[b, :k]
        assert got[2 * b + 1] == pytest.approx(float(xr @ xr), rel=1e-6)
        assert got[2 * b] == pytest.approx(float(rr @ rr), rel=1e-6)
    np.testing.assert_allclose(x.cpu().numpy(), xr, rtol=1e-6, atol=1e-5)
    np.testing.assert_allclose(r.cpu().numpy(), rr, rtol=1e-6, atol=1e-5)
    xs = x.cpu().numpy().astype(np.float64)
    assert got[2 * nb - 1] == pytest.approx(float(xs @ xs), rel=1e-12)


def test_reductions_are_bitwise_deterministic(cuda):
    torch = cuda
    L, k = 2086560, 20
    rng = np.random.default_rng(5)
    B = DeviceBasis(L, k + 2, torch.device("cuda", 0), torch)
    B.W[: k + 1, :L] = torch.from_numpy(rng.standard_normal((k + 1, L)).astype(np.float32)).cuda()
    v = torch.from_numpy(rng.standard_normal(L).astype(np.float32)).cuda()
    outs = []
    for _ in range(3):
        d = torch.zeros(k + 2, dtype=torch.float64, device="cuda")
        B.dots(k + 1, v, d, True, torch.cuda.current_stream())
        outs.append(d.cpu().numpy())
    assert all(np.array_equal(outs[0], o) for o in outs[1:])


@pytest.mark.parametrize("L,k", [(2086560, 30), (65536, 20)])
def test_single_pass_gram_schmidt(cuda, L, k):
    """reorthogonalize=False: one classical pass (streamed and SMEM paths)."""
    torch = cuda
    rng = np.random.default_rng(k)
    Q, _ = np.linalg.qr(rng.standard_normal((L, k + 1)))
    Q = Q.astype(np.float32).astype(np.float64)
    q = rng.standard_normal(L).astype(np.float32).astype(np.float64)
    B = basis_with(torch, Q, k + 3)
    qd = torch.from_numpy(q.astype(np.float32)).cuda()
    h = torch.zeros(k + 8, dtype=torch.float64, device="cuda")
    stat = torch.zeros(4, dtype=torch.float64, device="cuda")
    B.gs_step(k, qd, 1, h, stat, torch.cuda.current_stream())
    torch.cuda.synchronize()
    c = Q.T @ q
    v = q - Q @ c
    hg = h.cpu().numpy()[: k + 2]
    np.testing.assert_allclose(hg[: k + 1], c, rtol=1e-5, atol=1e-6 * np.abs(c).max())
    assert hg[k + 1] == pytest.approx(np.linalg.norm(v), rel=1e-5)
    w = B.W[k + 1, :L].cpu().numpy().astype(np.float64)
    np.testing.assert_allclose(w, v / np.linalg.norm(v), atol=2e-6)


# ---- the reference's step-wise API: ArnoldiState / arnoldi_step (row b seam)

def _ref_arnoldi(Mdense, r0, steps):
    """fp64 MGS + reorthogonalisation, ctkrylov/arnoldi.py:56-82 restated."""
    beta = np.linalg.norm(r0)
    V = [r0 / beta]
    cols = []
    for k in range(steps):
        q = Mdense @ V[k]
        h = np.zeros(k + 2)
        for _ in range(2):
            for i in range(k + 1):
                c = V[i] @ q
                h[i] += c
                q = q - c * V[i]
        h[k + 1] = np.linalg.norm(q)
        cols.append(h)
        V.append(q / h[k + 1])
    return beta, cols, V


def test_arnoldi_step_on_ct_composite(cuda):
    """compose(A, B) of GPU projectors runs on the device; the factorisation
    matches the fp64 reference Arnoldi and M W_k = W_{k+1} H_k."""
    from oracle import oracle as O
    from paper_2602_17892_b200 import arnoldi, ct, linop
    N, na, D = 24, 18, 35
    grid = ct.ImageGrid(N, N, 1.0)
    geom = ct.ParallelGeometry(np.arange(na) * np.pi / na, D, 1.0)
    A, B = ct.forward_ray_driven(grid, geom), ct.back_pixel_driven(grid, geom)
    M = linop.compose(A, B)                       # AB: m x m, applies on the device
    assert hasattr(M, "apply_device")
    og = O.Geometry(N, N, 1.0, geom.angles, D, 1.0)
    Ad = np.column_stack([O.forward(og, e) for e in np.eye(grid.n)])
    Bd = np.column_stack([O.back(og, e) for e in np.eye(geom.m)])
    r0 = np.random.default_rng(0).random(geom.m).astype(np.float32).astype(np.float64)
    st = arnoldi.ArnoldiState.start(r0, capacity=3)          # grows past its first rows
    steps = 8
    for _ in range(steps):
        arnoldi.arnoldi_step(st, M)
    beta, cols, V = _ref_arnoldi(Ad @ Bd, r0, steps)
    assert st.beta == pytest.approx(beta, rel=1e-12)
    H = st.hess
    Href = np.zeros((steps + 1, steps))
    for j, c in enumerate(cols):
        Href[: j + 2, j] = c
    np.testing.assert_allclose(H, Href, rtol=2e-4, atol=2e-4 * np.abs(Href).max())
    W = np.column_stack(st.basis)
    assert W.shape == (geom.m, steps + 1)
    assert np.abs(W.T @ W - np.eye(steps + 1)).max() < 1e-5
    resid = (Ad @ Bd) @ W[:, :steps] - W @ H
    assert np.linalg.norm(resid) <= 1e-4 * np.linalg.norm(H)


def test_arnoldi_step_host_operator_and_breakdown(cuda):
    """A host (dense) operator goes through its apply; an invariant subspace
    raises Breakdown(k) after recording the column, without a new row."""
    from paper_2602_17892_b200 import arnoldi, linop
    M = linop.dense_operator(np.diag([1.0, 2.0, 3.0, 4.0, 5.0, 6.0]))
    r0 = np.array([1.0, 1.0, 0.0, 0.0, 0.0, 0.0])           # spans a 2-D invariant subspace
    st = arnoldi.ArnoldiState.start(r0)
    arnoldi.arnoldi_step(st, M)
    with pytest.raises(arnoldi.Breakdown) as e:
        arnoldi.arnoldi_step(st, M)
    assert e.value.k == 2 and st.k == 2
    assert len(st.basis) == 2 and st.hess.shape == (3, 2)
    with pytest.raises(ValueError):
        arnoldi.ArnoldiState.start(np.zeros(4))
    st2 = arnoldi.ArnoldiState.start(np.ones(6))
    arnoldi.arnoldi_step(st2, M, reorthogonalize=False)
    assert st2.k == 1 and len(st2.basis) == 2


@pytest.mark.parametrize("seed", range(6))
def test_gram_schmidt_chains_random_lengths(cuda, seed):
    """Seeded random vector lengths from 2 to 3e6 (odd, prime-ish, around the
    path switches: fused / SMEM-resident / streamed, 128- and 256-float tiles,
    ragged last tiles) and chain lengths: every step of a chain on one basis
    against fp64 MGS + reorthogonalisation on the stored rows."""
    torch = cuda
    rng = np.random.default_rng(500 + seed)
    pool = [2, 3, 5, 17, 63, 64, 65, 255, 257, 1000, 4099, 32941, 65537, 151553, 151556,
            151808, 262147, 600001, 1000003, 2086561, 3000017]
    for _ in range(4):
        L = int(rng.choice(pool))
        K = int(min(L - 1, rng.integers(1, 12) if L > 300000 else rng.integers(1, 40)))
        if K < 1:
            continue
        B = DeviceBasis(L, K + 2, torch.device("cuda", 0), torch)
        v0 = rng.standard_normal(L)
        B.W[0, :L] = torch.from_numpy((v0 / np.linalg.norm(v0)).astype(np.float32)).cuda()
        st = torch.cuda.current_stream()
        h = torch.zeros(K + 8, dtype=torch.float64, device="cuda")
        stat = torch.zeros(4, dtype=torch.float64, device="cuda")
        for k in range(K):
            Q = B.W[: k + 1, :L].cpu().numpy().astype(np.float64).T
            q = (rng.standard_normal(L) + Q @ rng.standard_normal(k + 1)).astype(np.float32)
            B.cgs2_step(k, torch.from_numpy(q).cuda(), h, stat, st)
            torch.cuda.synchronize()
            href, v = mgs2_ref(Q, q.astype(np.float64))
            hg = h.cpu().numpy()[: k + 2]
            assert np.abs(hg - href).max() <= 1e-5 * np.abs(href).max(), (L, K, k)
            w = B.W[k + 1, :L].cpu().numpy().astype(np.float64)
            assert np.abs(w - v / href[k + 1]).max() < 5e-6, (L, K, k)
        W = B.W[: K + 1, :L].cpu().numpy().astype(np.float64)
        G = W @ W.T
        assert np.abs(G - np.eye(K + 1)).max() < 3e-6, (L, K)
