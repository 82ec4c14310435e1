"""Self-validation of the 3D extension of the oracle (oracle/refcpu/fem3d.hpp).

The reference is 2D only, so BASELINE configs 2 and 4 have no
reference arithmetic: parity is UNPINNED for them. These tests pin the 3D CPU
restatement by the properties a correct dQ1-SIPG / RT0 / dQ0 discretisation on
hexahedra must have; the device 3D assembly is then checked bit for bit against
it (tests/test_gpu_3d.py)."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import refcpu

TAGS3 = refcpu.TAGS3


def spec3(nx, ny, nz, lx=1.0, ly=1.0, lz=1.0, disp=None, flow=None, lam=2.0, mu=1.5, k_cells=None, **kw):
    disp = disp or {t: ("traction", (0.0, 0.0, 0.0)) for t in TAGS3}
    flow = flow or {t: ("pressure", 0.0) for t in TAGS3}
    d = dict(nx=nx, ny=ny, nz=nz, lx=lx, ly=ly, lz=lz, lam=lam, mu=mu, k_perm=1.0, eta=1.0, biot_m=10.0, biot_b=0.8,
             penalty=10.0, k_perm_cells=k_cells, disp=disp, flow=flow)
    d.update(kw)
    return d


def csr(rp, name, shape):
    off, idx, val = rp.csr(name)
    return sp.csr_matrix((val, idx, off), shape=shape)


def nodal_field(spec, fn):
    """dQ1 nodal interpolant of fn(x, y, z) -> (3,), dof = 24 c + 3 a + comp, a = 4 az + 2 ay + ax."""
    nx, ny, nz = spec["nx"], spec["ny"], spec["nz"]
    hx, hy, hz = spec["lx"] / nx, spec["ly"] / ny, spec["lz"] / nz
    u = np.zeros(24 * nx * ny * nz)
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                c = (k * ny + j) * nx + i
                for a in range(8):
                    ax, ay, az = a & 1, (a >> 1) & 1, a >> 2
                    u[24 * c + 3 * a:24 * c + 3 * a + 3] = fn((i + ax) * hx, (j + ay) * hy, (k + az) * hz)
    return u


def test_sizes_and_symmetry():
    s = spec3(3, 2, 4, lx=1.5, ly=1.0, lz=2.0)
    rp = refcpu.RefProblem(s)
    n = 3 * 2 * 4
    assert (rp.n_u, rp.n_p) == (24 * n, n)
    assert rp.n_q == 3 * 2 * 5 + 3 * 3 * 4 + 4 * 2 * 4
    A = csr(rp, "A", (rp.n_u, rp.n_u))
    assert abs(A - A.T).max() <= 1e-12 * abs(A).max()
    # every row of a cell couples to the cell and its face neighbours, 24 columns each
    off = rp.csr("A")[0]
    lens = np.diff(off).reshape(n, 24)
    assert (lens == lens[:, :1]).all() and set(np.unique(lens // 24)) <= {4, 5, 6, 7}
    Mq = csr(rp, "M_q", (rp.n_q, rp.n_q))
    assert abs(Mq - Mq.T).max() <= 1e-14
    mp = rp.misc()["m_p_diag"]
    assert np.allclose(mp, (1.5 / 3) * (1.0 / 2) * (2.0 / 4), rtol=1e-15)
    assert rp.misc()["k_dr"] == pytest.approx(2.0 + 2.0 * 1.5 / 3.0, rel=1e-15)


def test_rigid_body_modes_in_the_null_space():
    s = spec3(3, 3, 2, lx=1.0, ly=1.2, lz=0.7)
    rp = refcpu.RefProblem(s)
    A = csr(rp, "A", (rp.n_u, rp.n_u))
    scale = abs(A).max()
    modes = [lambda x, y, z: (1.0, 0.0, 0.0), lambda x, y, z: (0.0, 1.0, 0.0), lambda x, y, z: (0.0, 0.0, 1.0),
             lambda x, y, z: (-y, x, 0.0), lambda x, y, z: (0.0, -z, y), lambda x, y, z: (z, 0.0, -x)]
    for m in modes:
        u = nodal_field(s, m)
        assert abs(A @ u).max() <= 1e-11 * scale * abs(u).max()
    # and nothing else: with one fixed face the matrix is positive definite
    disp = {t: ("traction", (0.0, 0.0, 0.0)) for t in TAGS3}
    disp["zlo"] = ("fixed", (0.0, 0.0, 0.0))
    rp2 = refcpu.RefProblem(spec3(3, 3, 2, lx=1.0, ly=1.2, lz=0.7, disp=disp))
    A2 = csr(rp2, "A", (rp2.n_u, rp2.n_u)).toarray()
    w = np.linalg.eigvalsh(0.5 * (A2 + A2.T))
    assert w[0] > 1e-6 * w[-1]
    wn = np.linalg.eigvalsh(0.5 * (A.toarray() + A.toarray().T))
    assert (abs(wn[:6]) <= 1e-10 * wn[-1]).all() and wn[6] > 1e-6 * wn[-1]


def test_patch_test_constant_strain():
    """a(u_lin, v) = int_{boundary} (sigma n) . v for a globally linear u (no jumps, div sigma = 0): the cell
    term, the face consistency term and the traction load of assemble_rhs3 agree."""
    lam, mu = 2.0, 1.5
    G = np.array([[0.3, -0.2, 0.5], [0.1, 0.4, -0.6], [-0.7, 0.25, 0.15]])
    eps = 0.5 * (G + G.T)
    sig = 2 * mu * eps + lam * np.trace(eps) * np.eye(3)
    normals = {"xlo": (-1, 0, 0), "xhi": (1, 0, 0), "ylo": (0, -1, 0), "yhi": (0, 1, 0), "zlo": (0, 0, -1),
               "zhi": (0, 0, 1)}
    disp = {t: ("traction", tuple(sig @ np.array(nv, float))) for t, nv in normals.items()}
    s = spec3(3, 2, 3, lx=0.9, ly=1.1, lz=1.3, disp=disp, lam=lam, mu=mu)
    rp = refcpu.RefProblem(s)
    A = csr(rp, "A", (rp.n_u, rp.n_u))
    u = nodal_field(s, lambda x, y, z: tuple(G @ np.array([x, y, z]) + np.array([0.2, -0.1, 0.05])))
    ru, rq, rpp = rp.assemble_rhs(0.0)
    assert abs(A @ u - ru).max() <= 1e-11 * abs(ru).max()
    # divergence identity: (E^T u)_c = int_c div u for a continuous field
    E = csr(rp, "E", (rp.n_u, rp.n_p))
    vol = (0.9 / 3) * (1.1 / 2) * (1.3 / 3)
    assert np.allclose(E.T @ u, np.trace(G) * vol, rtol=1e-11)
    assert abs(rq).max() == 0.0 and abs(rpp).max() == 0.0


def test_uniaxial_compression_is_reproduced_exactly():
    """Fixed bottom, rollers on the sides, unit load on top: u = (0, 0, -z / (lambda + 2 mu)) is linear, and
    the Nitsche form is consistent, so the discrete solution equals it."""
    lam, mu = 2.0, 1.5
    disp = {"xlo": ("roller_x", (0, 0, 0)), "xhi": ("roller_x", (0, 0, 0)), "ylo": ("roller_y", (0, 0, 0)),
            "yhi": ("roller_y", (0, 0, 0)), "zlo": ("fixed", (0, 0, 0)), "zhi": ("traction", (0.0, 0.0, -1.0))}
    s = spec3(2, 3, 3, lx=1.0, ly=0.8, lz=1.5, disp=disp, lam=lam, mu=mu)
    rp = refcpu.RefProblem(s)
    A = csr(rp, "A", (rp.n_u, rp.n_u)).toarray()
    ru = rp.assemble_rhs(0.0)[0]
    u = np.linalg.solve(A, ru)
    ex = nodal_field(s, lambda x, y, z: (0.0, 0.0, -z / (lam + 2 * mu)))
    assert abs(u - ex).max() <= 1e-10 * abs(ex).max()
    # Dirichlet data: lift the bottom by a constant; the solution shifts rigidly
    disp["zlo"] = ("fixed", (0.0, 0.0, 0.25))
    rp2 = refcpu.RefProblem(spec3(2, 3, 3, lx=1.0, ly=0.8, lz=1.5, disp=disp, lam=lam, mu=mu))
    u2 = np.linalg.solve(csr(rp2, "A", (rp2.n_u, rp2.n_u)).toarray(), rp2.assemble_rhs(0.0)[0])
    assert abs(u2 - (ex + nodal_field(s, lambda x, y, z: (0.0, 0.0, 0.25)))).max() <= 1e-10


def test_flux_blocks():
    nx, ny, nz = 3, 2, 2
    lx, ly, lz = 1.2, 1.0, 0.8
    s = spec3(nx, ny, nz, lx=lx, ly=ly, lz=lz)
    rp = refcpu.RefProblem(s)
    Mq = csr(rp, "M_q", (rp.n_q, rp.n_q))
    B = csr(rp, "B", (rp.n_q, rp.n_p))
    hx, hy, hz = lx / nx, ly / ny, lz / nz
    nzf, nyf = nx * ny * (nz + 1), nx * (ny + 1) * nz

    def flux_of(v):  # q_f = v(face centre) . n_f, n_f the stored normal (outward on the boundary)
        q = np.zeros(rp.n_q)
        for k in range(nz + 1):
            for j in range(ny):
                for i in range(nx):
                    n = -1.0 if k == 0 else 1.0
                    q[(k * ny + j) * nx + i] = n * v((i + .5) * hx, (j + .5) * hy, k * hz)[2]
        for j in range(ny + 1):
            for k in range(nz):
                for i in range(nx):
                    n = -1.0 if j == 0 else 1.0
                    q[nzf + (j * nz + k) * nx + i] = n * v((i + .5) * hx, j * hy, (k + .5) * hz)[1]
        for i in range(nx + 1):
            for k in range(nz):
                for j in range(ny):
                    n = -1.0 if i == 0 else 1.0
                    q[nzf + nyf + (i * nz + k) * ny + j] = n * v(i * hx, (j + .5) * hy, (k + .5) * hz)[0]
        return q

    vol = hx * hy * hz
    qc = flux_of(lambda x, y, z: (0.7, -0.3, 0.2))
    assert abs(B.T @ qc).max() <= 1e-14                      # div of a constant field
    assert qc @ (Mq @ qc) == pytest.approx((0.49 + 0.09 + 0.04) * lx * ly * lz, rel=1e-13)
    ql = flux_of(lambda x, y, z: (x, 2 * y, -0.5 * z))
    assert np.allclose(B.T @ ql, -(1 + 2 - 0.5) * vol, rtol=1e-13)  # B^T q = -int div v
    # per-cell permeability scales the cell's mass contribution by eta / K_c
    k_cells = np.linspace(0.5, 2.0, nx * ny * nz)
    rp2 = refcpu.RefProblem(spec3(nx, ny, nz, lx=lx, ly=ly, lz=lz, k_cells=k_cells))
    Mq2 = csr(rp2, "M_q", (rp2.n_q, rp2.n_q))
    f = nzf + nyf + (1 * nz + 0) * ny + 0   # interior x face between cells (0,0,0) and (1,0,0)
    assert Mq2[f, f] == pytest.approx(vol / 3 * (1 / k_cells[0] + 1 / k_cells[1]), rel=1e-14)
    # no-flow faces are eliminated: identity rows, no B entries
    flow = {t: ("no_flow", 0.0) for t in TAGS3}
    flow["zhi"] = ("pressure", 0.0)
    rp3 = refcpu.RefProblem(spec3(nx, ny, nz, flow=flow))
    qcn = rp3.misc()["q_constrained"].astype(bool)
    assert qcn.sum() == 2 * (ny * nz + nx * nz) + nx * ny
    Mq3 = csr(rp3, "M_q", (rp3.n_q, rp3.n_q)).toarray()
    B3 = csr(rp3, "B", (rp3.n_q, rp3.n_p)).toarray()
    assert (Mq3[qcn] == np.eye(rp3.n_q)[qcn]).all() and (Mq3[:, qcn] == np.eye(rp3.n_q)[:, qcn]).all()
    assert abs(B3[qcn]).max() == 0.0


def test_config2_type_march_converges_and_conserves_mass():
    """dG(0) march of a small config-2-type problem through the oracle's solver stack (dense and banded
    inner solves agree); the per-cell discrete mass balance closes."""
    from paper_1801_04984_b200 import problem as P
    spec = P.config2(4).to_dict()
    rp = refcpu.RefProblem(spec)
    a = rp.march(0, 0.3, 3, tol=1e-10, restart=50, backend=0, keep_states=True)
    b = rp.march(0, 0.3, 3, tol=1e-10, restart=50, backend=1, keep_states=True)
    assert (a["iterations"] == b["iterations"]).all() and (a["iterations"] <= 12).all()
    for s in range(3):
        d = np.linalg.norm(a["states"][s] - b["states"][s]) / np.linalg.norm(a["states"][s])
        assert d <= 1e-9
    u_prev, p_prev = np.zeros(rp.n_u), np.zeros(rp.n_p)
    for s in range(3):
        rhs = rp.slab_rhs(0, 0.1 * s, 0.1, u_prev, p_prev)
        res, scale = rp.mass_residual(0, 0.1, rhs, a["states"][s].ravel())
        assert res.max() <= 1e-9 * scale
        st = a["states"][s][-1]
        u_prev, p_prev = st[:rp.n_u], st[rp.n_u + rp.n_q:]
    # the column settles: top displacement is downwards, pressure positive below the drained top
    uz_top = a["states"][-1][-1][:rp.n_u].reshape(-1, 8, 3)[-16:, 4:, 2]
    assert (uz_top < 0).all()


def test_config2_small_golden():
    """The committed fixture tests/golden/config2_small_oracle.npz (tests/golden/make_golden.py): the
    3D restatement reproduces its recorded operator sums, right-hand side, iteration counts and slab
    states for config 2 at 4^3, so an accidental edit of fem3d.hpp shows up here."""
    import os
    from paper_1801_04984_b200 import problem as P
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "config2_small_oracle.npz"))
    spec = P.config2(4)
    assert np.array_equal(spec.k_perm_cells, g["k_perm"])
    rp = refcpu.RefProblem(spec.to_dict())
    for nm in ("A", "M_q", "B", "E"):
        v = rp.csr(nm)[2]
        assert np.allclose([v.sum(), np.abs(v).sum()], g[f"sum_{nm}"], rtol=1e-13, atol=1e-9)
    ru, rq, rpp = rp.assemble_rhs(0.0)
    assert np.allclose([ru.sum(), rq.sum(), rpp.sum()], g["rhs_sums"], rtol=1e-13, atol=1e-15)
    res = rp.march(0, 0.3, 3, tol=1e-10, restart=50, backend=0, keep_states=True)
    assert np.array_equal(res["iterations"], g["iterations"])
    assert np.allclose(res["states"], g["states"], rtol=1e-11, atol=1e-16)


# ---- manufactured solutions: h-convergence of the 3D discretisation ----
def _mms_problem(n, disp_kinds, flow_kinds, lam=2.0, mu=1.5):
    disp = {t: (disp_kinds[t], (0.0, 0.0, 0.0)) for t in TAGS3}
    flow = {t: (flow_kinds[t], 0.0) for t in TAGS3}
    return spec3(n, n, n, disp=disp, flow=flow, lam=lam, mu=mu)


def _nodal_l2_error(spec, uh, exact):
    ue = nodal_field(spec, exact)
    return np.sqrt(np.mean((uh - ue) ** 2))


def test_mms_elasticity_second_order():
    """A u = f with a smooth manufactured displacement, Dirichlet (Nitsche) data on three faces and
    traction data on the other three, the body force f = -div sigma(u) and the boundary data sampled
    at the quadrature points (sympy): the nodal L2 error of the dQ1-SIPG solution drops with
    h^2 under refinement (n = 2, 4, 8), which a wrong cell term, face term, penalty or load would not."""
    import sympy as sy
    x, y, z = sy.symbols("x y z")
    lam, mu = 2.0, 1.5
    u = sy.Matrix([sy.sin(sy.pi * x) * sy.cos(sy.pi * y / 2) * (1 + z), x * y * sy.exp(-z) + sy.sin(y),
                   sy.cos(x) * z * z + x * y * z])
    grad = u.jacobian([x, y, z])
    eps = (grad + grad.T) / 2
    sig = 2 * mu * eps + lam * eps.trace() * sy.eye(3)
    f = -sy.Matrix([sum(sy.diff(sig[i, j], (x, y, z)[j]) for j in range(3)) for i in range(3)])
    u_f = sy.lambdify((x, y, z), u, "numpy")
    f_f = sy.lambdify((x, y, z), f, "numpy")
    sig_f = sy.lambdify((x, y, z), sig, "numpy")
    kinds = {"xlo": "fixed", "xhi": "traction", "ylo": "traction", "yhi": "fixed", "zlo": "fixed", "zhi": "traction"}
    normals = {1: (-1, 0, 0), 2: (1, 0, 0), 3: (0, -1, 0), 4: (0, 1, 0), 5: (0, 0, -1), 6: (0, 0, 1)}
    errs = []
    for n in (2, 4, 8):
        spec = _mms_problem(n, kinds, {t: "pressure" for t in TAGS3}, lam, mu)
        rp = refcpu.RefProblem(spec)
        cxyz, ids, fxyz = rp.sample_points3()
        mom = np.stack([np.broadcast_to(np.asarray(c, float), cxyz.shape[:2]) for c in
                        f_f(cxyz[..., 0], cxyz[..., 1], cxyz[..., 2])[:, 0]], axis=-1)
        X, Y, Z = fxyz[..., 0], fxyz[..., 1], fxyz[..., 2]
        uD = np.stack([np.broadcast_to(np.asarray(c, float), X.shape) for c in u_f(X, Y, Z)[:, 0]], axis=-1)
        S = sig_f(X, Y, Z)
        nx, ny, nz = n, n, n
        nzf, nyf = nx * ny * (nz + 1), nx * (ny + 1) * nz
        tags = np.array([(5 if f < nx * ny else 6) if f < nzf else
                         ((3 if (f - nzf) < nz * nx else 4) if f < nzf + nyf else
                          (1 if (f - nzf - nyf) < nz * ny else 2)) for f in ids])
        trac = np.zeros_like(uD)
        for b, tg in enumerate(tags):
            nv = np.array(normals[int(tg)], float)
            for i in range(3):
                trac[b, :, i] = sum(np.broadcast_to(np.asarray(S[i][j], float), X.shape)[b] * nv[j] for j in range(3))
        ru, rq, rpp = rp.rhs3_sampled(trac, uD, np.zeros(X.shape), momentum=mom)
        A = csr(rp, "A", (rp.n_u, rp.n_u)).tocsc()
        import scipy.sparse.linalg as spla
        uh = spla.spsolve(A, ru)
        errs.append(_nodal_l2_error(spec, uh, lambda a, b, c: np.asarray(u_f(a, b, c), float).ravel()))
    rates = [np.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert errs[2] < errs[1] < errs[0]
    assert rates[1] > 1.7, (errs, rates)


def test_mms_darcy_converges():
    """Mixed Darcy problem M_q q + B p = b_q, B^T q = b_p with K = 1: p = smooth field, q = -grad p,
    mass source g = div q, prescribed pressure on three faces and prescribed (nonzero) normal flux on
    the eliminated no-flow-kind faces: the cell-centre pressure error drops with h^2 (superconvergence
    of RT0 / dQ0 on uniform boxes) and the face fluxes converge, under n = 2, 4, 8."""
    import sympy as sy
    import scipy.sparse.linalg as spla
    x, y, z = sy.symbols("x y z")
    pex = sy.sin(sy.pi * x / 2) * sy.cos(y) * (1 + z * z) + x * y
    qex = -sy.Matrix([sy.diff(pex, v) for v in (x, y, z)])
    g = sum(sy.diff(qex[i], (x, y, z)[i]) for i in range(3))
    p_f, q_f, g_f = (sy.lambdify((x, y, z), e, "numpy") for e in (pex, qex, g))
    kinds = {"xlo": "pressure", "xhi": "no_flow", "ylo": "no_flow", "yhi": "pressure", "zlo": "no_flow", "zhi": "pressure"}
    normals = {1: (-1, 0, 0), 2: (1, 0, 0), 3: (0, -1, 0), 4: (0, 1, 0), 5: (0, 0, -1), 6: (0, 0, 1)}
    noflow_tags = {2, 3, 5}
    ep, eq = [], []
    for n in (2, 4, 8):
        spec = _mms_problem(n, {t: "traction" for t in TAGS3}, kinds)
        rp = refcpu.RefProblem(spec)
        cxyz, ids, fxyz = rp.sample_points3()
        mass = np.broadcast_to(np.asarray(g_f(cxyz[..., 0], cxyz[..., 1], cxyz[..., 2]), float), cxyz.shape[:2])
        X, Y, Z = fxyz[..., 0], fxyz[..., 1], fxyz[..., 2]
        nzf, nyf = n * n * (n + 1), n * (n + 1) * n
        tags = np.array([(5 if f < n * n else 6) if f < nzf else
                         ((3 if (f - nzf) < n * n else 4) if f < nzf + nyf else
                          (1 if (f - nzf - nyf) < n * n else 2)) for f in ids])
        Q = q_f(X, Y, Z)
        flow = np.broadcast_to(np.asarray(p_f(X, Y, Z), float), X.shape).copy()
        for b, tg in enumerate(tags):
            if int(tg) in noflow_tags:  # prescribed normal flux q . n
                nv = normals[int(tg)]
                flow[b] = sum(np.broadcast_to(np.asarray(Q[j][0], float), X.shape)[b] * nv[j] for j in range(3))
        zero3 = np.zeros(X.shape + (3,))
        ru, rq, rpp = rp.rhs3_sampled(zero3, zero3, flow, mass=mass)
        Mq, B = csr(rp, "M_q", (rp.n_q, rp.n_q)), csr(rp, "B", (rp.n_q, rp.n_p))
        K = sp.bmat([[Mq, B], [B.T, None]]).tocsc()
        sol = spla.spsolve(K, np.concatenate([rq, rpp]))
        qh, ph = sol[:rp.n_q], sol[rp.n_q:]
        h = 1.0 / n
        cc = np.array([((i + .5) * h, (j + .5) * h, (k + .5) * h) for k in range(n) for j in range(n) for i in range(n)])
        ep.append(np.sqrt(np.mean((ph - p_f(cc[:, 0], cc[:, 1], cc[:, 2])) ** 2)))
        # z-normal faces: q_f = q . n at the face centre, n the stored normal (outward on the boundary)
        fz = np.array([((i + .5) * h, (j + .5) * h, k * h, -1.0 if k == 0 else 1.0)
                       for k in range(n + 1) for j in range(n) for i in range(n)])
        qz = np.asarray(q_f(fz[:, 0], fz[:, 1], fz[:, 2])[2][0], float) * fz[:, 3]
        eq.append(np.sqrt(np.mean((qh[:nzf] - qz) ** 2)))
    assert np.log2(ep[1] / ep[2]) > 1.7, ep
    assert np.log2(eq[1] / eq[2]) > 0.9, eq
