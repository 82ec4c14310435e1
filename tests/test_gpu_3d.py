"""GPU tests of the 3D extension (BASELINE configs 2 / 4).

The reference is 2D only, so there is no reference arithmetic for
these configurations: PARITY UNPINNED. The checker is the 3D CPU restatement
oracle/refcpu/fem3d.hpp (pinned by its own properties, tests/test_oracle3d.py)
driving the same oracle solver stack as the 2D configurations. Bars: bit-exact
for the assembled operators, the right-hand side and the order-fixed SpMV;
GMRES iterations within +-1 and per-slab relative L2 <= 1e-9 for the solves;
at sizes the oracle cannot reach, the discrete mass balance and linearity."""
import numpy as np
import pytest

from paper_1801_04984_b200 import problem as P
from paper_1801_04984_b200 import solver as S

pytestmark = pytest.mark.gpu
SOLVE_RTOL = 1e-9


def _variants():
    out = []
    a = P.config2(3)
    a.nx, a.ny, a.nz = 3, 4, 2
    a.lx, a.ly, a.lz = 1.3, 0.9, 0.7
    a.k_perm_cells = P.lognormal_field(11, 24)
    out.append(a)
    b = P.config2(4)
    out.append(b)
    c = P.config2(3)
    c.nx, c.ny, c.nz = 2, 3, 3
    c.k_perm_cells = None
    c.disp = {"xlo": ("fixed", (0.1, 0.0, -0.2)), "xhi": ("roller_x", (0.0, 0.3, 0.1)),
              "ylo": ("roller_y", (0.2, 0.0, 0.4)), "yhi": ("traction", (0.1, -1.0, 0.5)),
              "zlo": ("roller_z", (0.3, -0.1, 0.0)), "zhi": ("fixed", (0.0, 0.0, 0.05))}
    c.flow = {"xlo": ("pressure", 0.5), "xhi": ("no_flow", 0.0), "ylo": ("no_flow", 0.0), "yhi": ("pressure", -0.25),
              "zlo": ("pressure", 0.0), "zhi": ("no_flow", 0.0)}
    out.append(c)
    d = P.config2(1)
    d.nx = d.ny = d.nz = 1
    d.k_perm_cells = None
    out.append(d)
    e = P.config2(5)
    e.nx, e.ny, e.nz = 5, 1, 2
    e.k_perm_cells = None
    e.disp = {t: ("fixed", (0.0, 0.0, 0.0)) for t in P.TAGS3}
    e.flow = {t: ("pressure", 0.0) for t in P.TAGS3}
    out.append(e)
    return out


@pytest.mark.parametrize("spec", _variants(), ids=lambda s: f"{s.nx}x{s.ny}x{s.nz}")
def test_device_assembly3_bit_identical(oracle, spec):
    """pdg_ops_assemble3 (one thread block per cell, one thread per face) == the 3D CPU
    restatement's triplet assembly merged in push order, bit for bit, and the constant-data
    right-hand side likewise."""
    rp = oracle.RefProblem(spec.to_dict())
    ops = S.SpatialOperators.assemble(spec)
    assert (ops.n_u, ops.n_q, ops.n_p) == (rp.n_u, rp.n_q, rp.n_p) == spec.sizes
    for name in ("A", "M_q", "B", "E"):
        ro, ri, rv = rp.csr(name)
        go, gi, gv = ops.download(name)
        assert np.array_equal(ro, go), name
        assert np.array_equal(ri, gi), name
        assert np.array_equal(rv, gv), name
    u, q, p = rp.assemble_rhs(0.3)
    gu, gq, gp = ops.rhs(0.3)
    assert np.array_equal(u, gu) and np.array_equal(q, gq) and np.array_equal(p, gp)


def test_device_assembly3_random_specs(oracle):
    """Seeded random 3D problems (mesh dimensions 1..4 per axis incl. single-cell directions, edge
    lengths, Lame parameters, penalty, per-cell permeability, every displacement / flow boundary
    kind with nonzero data): operators and right-hand side bit-identical to the CPU restatement."""
    rng = np.random.default_rng(20240611)
    kinds = ["fixed", "traction", "roller_x", "roller_y", "roller_z"]
    for case in range(12):
        nx, ny, nz = (int(v) for v in rng.integers(1, 5, 3))
        spec = P.config2(1)
        spec.nx, spec.ny, spec.nz = nx, ny, nz
        spec.lx, spec.ly, spec.lz = (float(v) for v in rng.uniform(0.5, 2.0, 3))
        spec.lam, spec.mu = float(rng.uniform(0.5, 5e3)), float(rng.uniform(0.5, 4e3))
        spec.penalty = float(rng.uniform(5.0, 40.0))
        spec.eta, spec.biot_m, spec.biot_b = float(rng.uniform(0.5, 2)), float(rng.uniform(1, 1e3)), float(rng.uniform(0.3, 1))
        spec.k_perm = float(rng.uniform(0.1, 3.0))
        spec.k_perm_cells = rng.lognormal(0.0, 1.0, nx * ny * nz) if case % 3 else None
        spec.disp = {t: (kinds[int(rng.integers(0, 5))], tuple(float(v) for v in rng.uniform(-1, 1, 3))) for t in P.TAGS3}
        spec.flow = {t: (("pressure", float(rng.uniform(-1, 1))) if rng.random() < 0.6 else ("no_flow", 0.0))
                     for t in P.TAGS3}
        rp = oracle.RefProblem(spec.to_dict())
        ops = S.SpatialOperators.assemble(spec)
        for name in ("A", "M_q", "B", "E"):
            ro, ri, rv = rp.csr(name)
            go, gi, gv = ops.download(name)
            assert np.array_equal(ro, go) and np.array_equal(ri, gi) and np.array_equal(rv, gv), (case, name)
        for a, b in zip(rp.assemble_rhs(0.1), ops.rhs(0.1)):
            assert np.array_equal(a, b), case


@pytest.mark.parametrize("r", [0, 1])
def test_spacetime_operator3_bit_identical(oracle, r):
    """Canonical space-time CSR of the 3D operators and its order-fixed SpMV == the oracle's
    canonical CSR and SparseMatrix::apply (sparse.hpp:30-40) on it, bit for bit."""
    spec = _variants()[0]
    rp = oracle.RefProblem(spec.to_dict())
    T = oracle.time_constants(r)["T"]
    tau = 0.1
    ops = S.SpatialOperators.assemble(spec)
    op = S.SpaceTimeOperator(ops, T, tau)
    ro, ri, rv = rp.spacetime_csr(T, tau)
    go, gi, gv = op.csr()
    assert np.array_equal(ro.astype(np.int64), go)
    assert np.array_equal(ri, gi)
    assert np.array_equal(rv, gv)
    import torch
    x = P.uniform_vector(P.X_SEED, op.rows)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    torch.cuda.synchronize()
    op.apply_device(xd.data_ptr(), yd.data_ptr())
    assert np.array_equal(yd.cpu().numpy(), oracle.csr_apply(ro, ri, rv, x))
    # matrix-free form of the reference (fixed_stress.hpp:38-60) on the 3D blocks: roundoff only
    y_mf = rp.apply_block(T, tau, x)
    assert np.linalg.norm(yd.cpu().numpy() - y_mf) <= 1e-12 * np.linalg.norm(y_mf)


def test_preconditioner3_matches_oracle(oracle):
    """One truncated fixed-stress sweep (fixed_stress.hpp:109-139) with the exact nested-dissection
    inner solves on the 3D operators against the oracle's dense-LU sweep; linear and repeatable."""
    spec = P.config2(4)
    rp = oracle.RefProblem(spec.to_dict())
    ops = S.SpatialOperators.assemble(spec)
    tau, lam = 0.1, 1.0
    blk = S.BlockSolver(ops, [[lam]], tau)
    r = P.uniform_vector(5, rp.n_total)
    z = blk.precondition(r)
    zr = rp.precondition(lam, tau, r, sweeps=1, backend=0)
    assert np.linalg.norm(z - zr) <= 1e-10 * np.linalg.norm(zr)
    assert np.array_equal(z, blk.precondition(r))
    r2 = P.uniform_vector(6, rp.n_total)
    lin = blk.precondition(2.0 * r - 3.0 * r2) - (2.0 * z - 3.0 * blk.precondition(r2))
    assert np.abs(lin).max() <= 1e-11 * np.abs(z).max()


@pytest.mark.parametrize("candidate", ["reference", "flexible"])
@pytest.mark.parametrize("n", [4, 6])
def test_march_config2_type_parity(oracle, n, candidate):
    """dG(0) march of config 2 at n^3 (layered permeability over 8 layers, fixed bottom, loaded
    drained top): GMRES iterations within +-1 of the oracle and per-slab relative L2 <= 1e-9."""
    spec = P.config2(n)
    rp = oracle.RefProblem(spec.to_dict())
    n_slabs = 3
    ref = rp.march(0, 0.3, n_slabs, tol=1e-10, restart=50, backend=1, flexible=candidate == "flexible",
                   keep_states=True)
    ops = S.SpatialOperators.assemble(spec)
    opt = S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=50), candidate=candidate)
    reps, states = S.march(ops, 0, 0.3, n_slabs, opt, keep_states=True, mass_check=True)
    for s in range(n_slabs):
        assert reps[s].converged
        assert abs(reps[s].iterations - int(ref["iterations"][s])) <= 1, (s, reps[s].iterations, ref["iterations"])
        d = np.linalg.norm(states[s] - ref["states"][s].ravel()) / np.linalg.norm(ref["states"][s])
        assert d <= SOLVE_RTOL, (s, d)
        assert reps[s].mass_rel <= 1e-9


@pytest.mark.parametrize("dim", [2, 3])
def test_nd_streaming_mode_matches_default(oracle, monkeypatch, dim):
    """The streaming mode of the nested-dissection solves (nd_stream.cu: postorder numeric
    factorization with one front matrix per pending update, one level kernel per depth and pass on
    the row-major factor; selected automatically for wide 3D fronts, forced here by
    PDG_ND_STREAM=1) is the same exact solve as the default kernels: preconditioner within
    roundoff, same GMRES iterations, solution within 1e-9 of the oracle."""
    spec = P.config1(32) if dim == 2 else P.config2(6)
    r = 1 if dim == 2 else 0
    rp = oracle.RefProblem(spec.to_dict())
    T = oracle.time_constants(r)["T"]
    tau = 0.05
    ops = S.SpatialOperators.assemble(spec)
    opt = S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=50), candidate="flexible")
    blk = S.BlockSolver(ops, T, tau, opt=opt)
    monkeypatch.setenv("PDG_ND_STREAM", "1")
    ops_s = S.SpatialOperators.assemble(spec)  # its own operators: the displacement factorization is cached per handle
    blk_s = S.BlockSolver(ops_s, T, tau, opt=opt)
    monkeypatch.delenv("PDG_ND_STREAM")
    rvec = P.uniform_vector(9, blk.rows)
    z, zs = blk.precondition(rvec), blk_s.precondition(rvec)
    assert np.linalg.norm(z - zs) <= 1e-11 * np.linalg.norm(z)
    assert np.array_equal(zs, blk_s.precondition(rvec))
    rhs = P.uniform_vector(10, blk.rows)
    x, rep = blk.solve(rhs)
    xs, reps = blk_s.solve(rhs)
    assert rep.iterations == reps.iterations
    assert np.linalg.norm(x - xs) <= 1e-9 * np.linalg.norm(x)
    xr, _ = rp.block_solve(r, tau, rhs, tol=1e-10, restart=50, backend=1, flexible=True)
    assert np.linalg.norm(xs - xr) <= SOLVE_RTOL * np.linalg.norm(xr)


@pytest.mark.parametrize("r", [0, 1])
def test_fast_mode_fp32_factor(oracle, monkeypatch, r):
    """pdg_gmres_opts.mode 1 (SURVEY 8(b) SolveOptions mode = fast): the streamed displacement factor
    stored in fp32, sums in fp64. The preconditioner differs from the exact one at the fp32 level
    (so the path really ran), GMRES reaches the same fp64 true-residual tolerance within one extra
    iteration, the solution is within 1e-8 of the parity mode's and of the oracle's, and repeats
    are bit-identical. Parity mode on the same operators is untouched (its own factorization)."""
    spec = P.config2(6)
    rp = oracle.RefProblem(spec.to_dict())
    T = oracle.time_constants(r)["T"]
    tau = 0.05
    monkeypatch.setenv("PDG_ND_STREAM", "1")
    ops = S.SpatialOperators.assemble(spec)
    par = S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=50), candidate="flexible")
    fast = S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=50), candidate="flexible", mode="fast")
    blk = S.BlockSolver(ops, T, tau, opt=par)
    blk_f = S.BlockSolver(ops, T, tau, opt=fast)
    monkeypatch.delenv("PDG_ND_STREAM")
    rvec = P.uniform_vector(9, blk.rows)
    z, zf = blk.precondition(rvec), blk_f.precondition(rvec)
    nu = ops.n_u  # the displacement part of component 0 (the flux and pressure parts do not use the factor)
    dz = np.linalg.norm(z[:nu] - zf[:nu]) / np.linalg.norm(z[:nu])
    assert 1e-10 < dz < 1e-5, dz  # fp32-stored factor: different from, and close to, the exact solve
    assert np.array_equal(zf, blk_f.precondition(rvec))
    assert np.array_equal(z, blk.precondition(rvec))
    rhs = P.uniform_vector(10, blk.rows)
    x, rep = blk.solve(rhs)
    xf, repf = blk_f.solve(rhs)
    assert repf.converged and repf.final_relative_residual <= 1e-10
    assert rep.iterations <= repf.iterations <= rep.iterations + 1, (rep.iterations, repf.iterations)
    assert np.linalg.norm(x - xf) <= 1e-8 * np.linalg.norm(x)
    xr, _ = rp.block_solve(r, tau, rhs, tol=1e-10, restart=50, backend=1, flexible=True)
    assert np.linalg.norm(xf - xr) <= 1e-8 * np.linalg.norm(xr)
    import ctypes as C
    from paper_1801_04984_b200 import _lib
    bad = par.to_struct()
    bad.mode = 7
    h = C.c_void_p()
    th = np.ones(1)
    with pytest.raises(_lib.InvalidArgument):
        _lib.check(_lib.lib().pdg_block_create(ops._h, 1, th.ctypes.data_as(_lib.DP), tau, 1.0, C.byref(bad), C.byref(h)))


@pytest.mark.parametrize("candidate", ["reference", "flexible"])
def test_march_3d_dg1_parity(oracle, candidate):
    """dG(1) in 3D (the element pair of config 4 at a size the oracle reaches, 4^3): the 2x2
    Schur block with two right-hand sides per inner solve; iterations within +-1, states within
    1e-9 of the oracle."""
    spec = P.config2(4)
    spec.k_perm_cells = P.lognormal_field(7, 64, 1.5)
    rp = oracle.RefProblem(spec.to_dict())
    ref = rp.march(1, 0.25, 2, tol=1e-10, restart=50, backend=1, flexible=candidate == "flexible", keep_states=True)
    ops = S.SpatialOperators.assemble(spec)
    opt = S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=50), candidate=candidate)
    reps, states = S.march(ops, 1, 0.25, 2, opt, keep_states=True, mass_check=True)
    for s in range(2):
        assert reps[s].converged
        assert abs(reps[s].iterations - int(ref["iterations"][s])) <= 1
        d = np.linalg.norm(states[s] - ref["states"][s].ravel()) / np.linalg.norm(ref["states"][s])
        assert d <= SOLVE_RTOL, (s, d)
        assert reps[s].mass_rel <= 1e-7


def test_fixed_stress_march_3d(oracle):
    """The fixed-stress branch of the march (march.hpp:80-108, dG(0)) on the 3D operators: sweep
    counts identical to the oracle's, states within 1e-8 (the iteration stops at tol 1e-10)."""
    spec = P.config2(4)
    rp = oracle.RefProblem(spec.to_dict())
    ref = rp.march_fs(0, 0.3, 3, tol=1e-10, backend=1, keep_states=True)
    ops = S.SpatialOperators.assemble(spec)
    reps, states = S.march(ops, 0, 0.3, 3, S.SolveOptions(), keep_states=True, method="fixed-stress")
    assert [r.iterations for r in reps] == [int(v) for v in ref["sweeps"]]
    for s in range(3):
        d = np.linalg.norm(states[s] - ref["states"][s].ravel()) / np.linalg.norm(ref["states"][s])
        assert d <= 1e-8, (s, d)


def test_upload3_matches_device_assembly(oracle):
    """Operators assembled by the CPU restatement and uploaded (pdg_ops_upload3) give the same
    slab solve, bit for bit, as the device-assembled ones."""
    spec = P.config2(4)
    rp = oracle.RefProblem(spec.to_dict())
    m = rp.misc()
    blocks = {k: rp.csr(k) for k in ("A", "M_q", "B", "E")}
    up = S.SpatialOperators.upload(spec.nx, spec.ny, blocks, m["m_p_diag"], m["q_constrained"], m["biot_b"],
                                   m["inv_m"], m["k_dr"], nz=spec.nz)
    dev = S.SpatialOperators.assemble(spec)
    opt = S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=50), candidate="flexible")
    rhs = rp.slab_rhs(0, 0.0, 0.1, np.zeros(rp.n_u), np.zeros(rp.n_p))
    xa, ra = S.SlabSolver(up, 0, 0.1, opt).solve(rhs)
    xb, rb = S.SlabSolver(dev, 0, 0.1, opt).solve(rhs)
    assert ra.iterations == rb.iterations and np.array_equal(xa, xb)
    with pytest.raises(S.InvalidArgument):
        S.SpatialOperators.upload(spec.nx, spec.ny, blocks, m["m_p_diag"], m["q_constrained"], m["biot_b"],
                                  m["inv_m"], m["k_dr"], nz=spec.nz + 1)


def test_march_config2_12cubed_properties():
    """Beyond the oracle's reach (12^3: 41,472 displacement dofs): every slab converges, the
    per-cell discrete mass balance closes (slab.hpp:292-318 on the device), the iteration count
    stays that of the small meshes, and repeats are bit-identical."""
    spec = P.config2(12)
    ops = S.SpatialOperators.assemble(spec)
    opt = S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=50), candidate="flexible")
    reps, states = S.march(ops, 0, 0.2, 2, opt, keep_states=True, mass_check=True)
    reps2, states2 = S.march(ops, 0, 0.2, 2, opt, keep_states=True)
    for s in range(2):
        assert reps[s].converged and reps[s].iterations <= 20
        assert reps[s].final_relative_residual <= 1e-10
        assert reps[s].mass_rel <= 1e-7  # GMRES tol 1e-10 times the conditioning (2D config 1 uses the same bar)
        assert np.array_equal(states[s], states2[s])
    nu = ops.n_u
    uz = states[-1][:nu].reshape(-1, 8, 3)[:, :, 2]
    assert uz.min() < 0.0 and uz.min() > -1.0  # the loaded top settles, by less than the domain height


def test_config2_full_size_32cubed():
    """BASELINE config 2 at its full size (32^3 hexahedra: 786,432 displacement dofs, ~80 GB of
    nested-dissection factors, streaming mode): the slabs converge in the iteration count of the
    small meshes (4), the true residual meets the tolerance, the per-cell mass balance closes,
    the SpMV is linear (A(2x) = 2 A x exactly) and the solve repeats bit for bit."""
    import torch
    spec = P.config2(32)
    ops = S.SpatialOperators.assemble(spec)
    assert (ops.n_u, ops.n_q, ops.n_p) == (786432, 101376, 32768)
    opt = S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=50), candidate="flexible")
    slab = S.SlabSolver(ops, 0, 0.1, opt)
    dev = torch.device("cuda")
    nt = ops.n_total
    u_prev = torch.zeros(ops.n_u, dtype=torch.float64, device=dev)
    p_prev = torch.zeros(ops.n_p, dtype=torch.float64, device=dev)
    rhs = torch.empty(nt, dtype=torch.float64, device=dev)
    out = torch.empty_like(rhs)
    out2 = torch.empty_like(rhs)
    res = torch.empty(ops.n_p, dtype=torch.float64, device=dev)
    for k in range(2):
        torch.cuda.synchronize()
        slab.rhs_device(0.1 * k, u_prev.data_ptr(), p_prev.data_ptr(), rhs.data_ptr())
        rep = slab.solve_device(rhs.data_ptr(), out.data_ptr())
        assert rep.converged and rep.iterations <= 6 and rep.final_relative_residual <= 1e-10
        scale = slab.mass_residual_device(rhs.data_ptr(), out.data_ptr(), res.data_ptr())
        assert float(res.max().item()) <= 1e-7 * scale
        rep2 = slab.solve_device(rhs.data_ptr(), out2.data_ptr())
        assert rep2.iterations == rep.iterations and torch.equal(out, out2)
        u_prev.copy_(out[:ops.n_u])
        p_prev.copy_(out[ops.n_u + ops.n_q:])
    uz = out[:ops.n_u].reshape(-1, 8, 3)[:, :, 2]
    assert float(uz.min()) < 0.0 and float(uz.min()) > -1.0
    del slab
    op = S.SpaceTimeOperator(ops, [[1.0]], 0.1)
    x = torch.from_numpy(P.uniform_vector(P.X_SEED, op.rows)).cuda()
    y, y2 = torch.empty_like(x), torch.empty_like(x)
    torch.cuda.synchronize()
    op.apply_device(x.data_ptr(), y.data_ptr())
    x2 = 2.0 * x
    torch.cuda.synchronize()
    op.apply_device(x2.data_ptr(), y2.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(y2, 2.0 * y)


def test_gpu_against_committed_golden_vectors():
    """The GPU march against the committed fixtures (no oracle call): config 2 at 4^3
    (tests/golden/config2_small_oracle.npz) and dG(2) / dG(3) at 6^2 (highorder_oracle.npz)."""
    import os
    golden = os.path.join(os.path.dirname(__file__), "golden")
    g = np.load(os.path.join(golden, "config2_small_oracle.npz"))
    opt = S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=50))
    ops = S.SpatialOperators.assemble(P.config2(4))
    reps, states = S.march(ops, 0, 0.3, 3, opt, keep_states=True)
    for s in range(3):
        assert abs(reps[s].iterations - int(g["iterations"][s])) <= 1
        ref = g["states"][s].ravel()
        assert np.linalg.norm(states[s] - ref) <= SOLVE_RTOL * np.linalg.norm(ref)
    h = np.load(os.path.join(golden, "highorder_oracle.npz"))
    spec = P.config0()
    spec.nx = spec.ny = 6
    ops2 = S.SpatialOperators.assemble(spec)
    for r in (2, 3):
        reps, states = S.march(ops2, r, 0.3, 2, opt, keep_states=True)
        for s in range(2):
            assert abs(reps[s].iterations - int(h[f"iterations_r{r}"][s])) <= 1
            ref = h[f"states_r{r}"][s].ravel()
            assert np.linalg.norm(states[s] - ref) <= SOLVE_RTOL * np.linalg.norm(ref)


def test_rhs_sampled3_bit_identical(oracle):
    """pdg_ops_rhs_sampled on 3D operators == the oracle's assemble_rhs3_sampled, bit for bit, for
    seeded random volume sources and boundary data (Dirichlet, traction, pressure and prescribed
    nonzero normal flux, eliminated couplings included); the library's sample points are the
    oracle's; absent volume fields are skipped; constant data through the sampled path equals the
    constant-data kernels."""
    spec = _variants()[2]  # every boundary kind
    rp = oracle.RefProblem(spec.to_dict())
    ops = S.SpatialOperators.assemble(spec)
    cxyz, ids, fxyz = rp.sample_points3()
    gc, gi, gf = ops.sample_points()
    assert np.array_equal(cxyz, gc) and np.array_equal(ids, gi) and np.array_equal(fxyz, gf)
    rng = np.random.default_rng(7)
    sm = dict(momentum=rng.standard_normal(cxyz.shape), darcy=rng.standard_normal(cxyz.shape),
              mass=rng.standard_normal(cxyz.shape[:2]), traction=rng.standard_normal(fxyz.shape),
              dirichlet=rng.standard_normal(fxyz.shape), flow=rng.standard_normal(fxyz.shape[:2]))
    for drop in ((), ("momentum",), ("darcy", "mass"), ("momentum", "darcy", "mass")):
        cur = {k: (None if k in drop else v) for k, v in sm.items()}
        ref = rp.rhs3_sampled(cur["traction"], cur["dirichlet"], cur["flow"], momentum=cur["momentum"],
                              darcy=cur["darcy"], mass=cur["mass"])
        got = ops.rhs_sampled(cur)
        for a, b in zip(ref, got):
            assert np.array_equal(a, b), drop
    # constant boundary data as samples == the constant-data right-hand side
    const = dict(traction=np.zeros(fxyz.shape), dirichlet=np.zeros(fxyz.shape), flow=np.zeros(fxyz.shape[:2]))
    nx, ny, nz = spec.nx, spec.ny, spec.nz
    nzf, nyf = nx * ny * (nz + 1), nx * (ny + 1) * nz
    for b, f in enumerate(ids):
        tag = (("zlo" if f < nx * ny else "zhi") if f < nzf else
               (("ylo" if f - nzf < nz * nx else "yhi") if f < nzf + nyf else ("xlo" if f - nzf - nyf < nz * ny else "xhi")))
        kind, data = spec.disp[tag]
        (const["dirichlet"] if kind == "fixed" else const["traction"])[b, :, :] = data
        const["flow"][b, :] = spec.flow[tag][1]
    for a, b in zip(ops.rhs(0.0), ops.rhs_sampled(const)):
        assert np.array_equal(a, b)


def test_mms_poroelastic_march_converges_on_device():
    """End-to-end manufactured solution of the coupled 3D Biot system on the GPU (device assembly,
    sampled time-dependent sources and boundary data, dG(1) slabs, GMRES with the exact fixed-stress
    preconditioner): u(x, t) = U(x)(1 + t), p(x, t) = P(x)(1 + t/2), q = -(K/eta) grad p, with
    f = -div(sigma(u) - b p I) and g = d/dt(b div u + p/M) + div q. The solution is linear in time, so
    dG(1) is exact in time and the error at the end of the march is the spatial one: second order in
    the nodal displacement, at least first order in the piecewise-constant pressure (measured:
    2.2 / 2.2 and 2.7 / 1.4 under n = 2, 4, 8). Parity is unpinned in 3D; this pins the whole device
    path against the continuous problem."""
    import sympy as sy
    import torch
    x, y, z, t = sy.symbols("x y z t")
    lam, mu, bb, MM, eta, kperm = 2.0, 1.5, 0.8, 10.0, 1.0, 1.0
    U = sy.Matrix([sy.sin(sy.pi * x / 2) * sy.cos(y) * (1 + z), x * y * sy.exp(-z), sy.cos(x) * z * z + x * y * z]) * sy.Rational(1, 10)
    P_ = sy.sin(sy.pi * x / 2) * sy.cos(y) * (1 + z * z) + x * y
    u = U * (1 + t)
    p = P_ * (1 + t / 2)
    grad = u.jacobian([x, y, z])
    eps = (grad + grad.T) / 2
    sig = 2 * mu * eps + lam * eps.trace() * sy.eye(3) - bb * p * sy.eye(3)
    fm = -sy.Matrix([sum(sy.diff(sig[i, j], (x, y, z)[j]) for j in range(3)) for i in range(3)])
    q = -(kperm / eta) * sy.Matrix([sy.diff(p, v) for v in (x, y, z)])
    g = sy.diff(bb * eps.trace() + p / MM, t) + sum(sy.diff(q[i], (x, y, z)[i]) for i in range(3))
    L = lambda e: sy.lambdify((x, y, z, t), e, "numpy")  # noqa: E731
    u_f, p_f, fm_f, g_f = L(u), L(p), L(fm), L(g)

    def vec(fn, X, Y, Z, tt):
        out = fn(X, Y, Z, tt)
        return np.stack([np.broadcast_to(np.asarray(out[i][0], float), X.shape) for i in range(3)], axis=-1)

    def sca(fn, X, Y, Z, tt):
        return np.broadcast_to(np.asarray(fn(X, Y, Z, tt), float), X.shape).copy()

    r, n_slabs, T = 1, 2, 0.5
    tau = T / n_slabs
    nodes = S.time_constants(r)["nodes"]
    opt = S.SolveOptions(gmres=S.GmresOptions(tol=1e-12, restart=50), candidate="flexible")
    eu, ep = [], []
    for n in (2, 4, 8):
        spec = P.config2(n)
        spec.lam, spec.mu, spec.biot_b, spec.biot_m, spec.eta, spec.k_perm = lam, mu, bb, MM, eta, kperm
        spec.k_perm_cells = None
        spec.disp = {tg: ("fixed", (0.0, 0.0, 0.0)) for tg in P.TAGS3}
        spec.flow = {tg: ("pressure", 0.0) for tg in P.TAGS3}
        ops = S.SpatialOperators.assemble(spec)
        cxyz, ids, fxyz = ops.sample_points()
        h = 1.0 / n
        # initial data: nodal interpolant of u(0), cell-centre value of p(0)
        nod = np.array([[((i + (a & 1)) * h, (j + ((a >> 1) & 1)) * h, (k + (a >> 2)) * h) for a in range(8)]
                        for k in range(n) for j in range(n) for i in range(n)])
        cc = np.array([((i + .5) * h, (j + .5) * h, (k + .5) * h) for k in range(n) for j in range(n) for i in range(n)])
        u_prev = torch.from_numpy(vec(u_f, nod[..., 0], nod[..., 1], nod[..., 2], 0.0).reshape(-1).copy()).cuda()
        p_prev = torch.from_numpy(sca(p_f, cc[:, 0], cc[:, 1], cc[:, 2], 0.0)).cuda()
        slab = S.SlabSolver(ops, r, tau, opt)
        nt = ops.n_total
        rhs = torch.empty((r + 1) * nt, dtype=torch.float64, device="cuda")
        out = torch.empty_like(rhs)
        for s_ in range(n_slabs):
            t0 = s_ * tau
            samples = []
            for c in nodes:
                tt = t0 + c * tau
                samples.append(dict(
                    momentum=vec(fm_f, cxyz[..., 0], cxyz[..., 1], cxyz[..., 2], tt),
                    mass=sca(g_f, cxyz[..., 0], cxyz[..., 1], cxyz[..., 2], tt),
                    traction=np.zeros(fxyz.shape), dirichlet=vec(u_f, fxyz[..., 0], fxyz[..., 1], fxyz[..., 2], tt),
                    flow=sca(p_f, fxyz[..., 0], fxyz[..., 1], fxyz[..., 2], tt)))
            torch.cuda.synchronize()
            slab.rhs_sampled_device(samples, u_prev.data_ptr(), p_prev.data_ptr(), rhs.data_ptr())
            rep = slab.solve_device(rhs.data_ptr(), out.data_ptr())
            assert rep.converged
            end = out[r * nt:(r + 1) * nt]
            u_prev.copy_(end[:ops.n_u])
            p_prev.copy_(end[ops.n_u + ops.n_q:])
            torch.cuda.synchronize()
        ue = vec(u_f, nod[..., 0], nod[..., 1], nod[..., 2], T).reshape(-1)
        pe = sca(p_f, cc[:, 0], cc[:, 1], cc[:, 2], T)
        eu.append(float(np.sqrt(np.mean((u_prev.cpu().numpy() - ue) ** 2))))
        ep.append(float(np.sqrt(np.mean((p_prev.cpu().numpy() - pe) ** 2))))
    ru = [np.log2(eu[i] / eu[i + 1]) for i in range(2)]
    rp_ = [np.log2(ep[i] / ep[i + 1]) for i in range(2)]
    print("MMS 3D march: u errors", eu, "rates", ru, "p errors", ep, "rates", rp_)
    assert eu[2] < eu[1] < eu[0] and ep[2] < ep[1] < ep[0]
    assert ru[1] > 1.7 and rp_[1] > 0.9, (eu, ru, ep, rp_)
