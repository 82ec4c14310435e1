"""GPU parity tests: the CUDA path (through the C ABI) against the CPU oracle
on the same seeded inputs. Bars: bit-exact for the assembled operators and the
order-fixed SpMV; GMRES iterations within +-1 and per-slab relative L2
difference <= 1e-9 for the solves (BASELINE.json north_star)."""
import json
import os

import numpy as np
import pytest

from paper_1801_04984_b200 import problem as P
from paper_1801_04984_b200 import solver as S

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
SOLVE_RTOL = 1e-9  # per-slab relative L2 (north_star)


def _bc_variants():
    """Boundary combinations covering every Nitsche / flux branch of the assembly."""
    out = []
    a = P.config0()
    a.nx, a.ny = 5, 3
    out.append(a)
    b = P.terzaghi_recorded()
    out.append(b)
    c = P.config1(6)
    c.disp = {"left": ("fixed", (0.0, 0.0)), "right": ("roller_x", (0.0, 0.3)),
              "bottom": ("roller_y", (0.2, 0.0)), "top": ("traction", (0.1, -1.0))}
    c.flow = {"left": ("pressure", 0.5), "right": ("no_flow", 0.0), "bottom": ("no_flow", 0.0),
              "top": ("pressure", -0.25)}
    c.lx, c.ly = 1.3, 0.9
    out.append(c)
    d = P.config0()
    d.nx, d.ny = 7, 4
    d.disp = {t: ("fixed", (0.0, 0.0)) for t in P.TAGS}
    d.flow = {t: ("pressure", 0.0) for t in P.TAGS}
    out.append(d)
    out.append(P.config1(32))
    return out


@pytest.mark.parametrize("spec", _bc_variants(), ids=lambda s: f"{s.nx}x{s.ny}")
def test_device_assembly_bit_identical(oracle, spec):
    """pdg_ops_assemble (one thread block per cell) == assemble_operators +
    csr_from_triplets (assembly.hpp:177-395, sparse.hpp:83-110), bit for bit."""
    rp = oracle.RefProblem(spec.to_dict())
    ops = S.SpatialOperators.assemble(spec)
    for name in ("A", "M_q", "B", "E"):
        ro, ri, rv = rp.csr(name)
        go, gi, gv = ops.download(name)
        assert np.array_equal(ro, go), name
        assert np.array_equal(ri, gi), name
        assert np.array_equal(rv, gv), name  # exact (== treats +0/-0 alike)
    u, q, p = rp.assemble_rhs(0.3)
    gu, gq, gp = ops.rhs(0.3)
    assert np.array_equal(u, gu) and np.array_equal(q, gq) and np.array_equal(p, gp)


def test_device_assembly_random_specs(oracle):
    """Seeded random 2D problems (mesh dimensions 1..7, edge lengths, material, penalty, per-cell
    permeability, every boundary kind with nonzero data): bit-identical operators and rhs."""
    rng = np.random.default_rng(1801)
    kinds = ["fixed", "traction", "roller_x", "roller_y"]
    for case in range(16):
        spec = P.config0()
        spec.nx, spec.ny = (int(v) for v in rng.integers(1, 8, 2))
        spec.lx, spec.ly = (float(v) for v in rng.uniform(0.5, 2.0, 2))
        spec.lam, spec.mu = float(rng.uniform(0.5, 5e3)), float(rng.uniform(0.5, 4e3))
        spec.penalty = float(rng.uniform(5.0, 40.0))
        spec.eta, spec.biot_m, spec.biot_b = float(rng.uniform(0.5, 2)), float(rng.uniform(1, 1e3)), float(rng.uniform(0.3, 1))
        spec.k_perm = float(rng.uniform(0.1, 3.0))
        spec.k_perm_cells = rng.lognormal(0.0, 1.0, spec.nx * spec.ny) if case % 3 else None
        spec.disp = {t: (kinds[int(rng.integers(0, 4))], tuple(float(v) for v in rng.uniform(-1, 1, 2))) for t in P.TAGS}
        spec.flow = {t: (("pressure", float(rng.uniform(-1, 1))) if rng.random() < 0.6 else ("no_flow", 0.0))
                     for t in P.TAGS}
        rp = oracle.RefProblem(spec.to_dict())
        ops = S.SpatialOperators.assemble(spec)
        for name in ("A", "M_q", "B", "E"):
            ro, ri, rv = rp.csr(name)
            go, gi, gv = ops.download(name)
            assert np.array_equal(ro, go) and np.array_equal(ri, gi) and np.array_equal(rv, gv), (case, name)
        for a, b in zip(rp.assemble_rhs(0.1), ops.rhs(0.1)):
            assert np.array_equal(a, b), case


def _upload_from_oracle(rp, spec):
    m = rp.misc()
    blocks = {k: rp.csr(k) for k in ("A", "M_q", "B", "E")}
    return S.SpatialOperators.upload(spec.nx, spec.ny, blocks, m["m_p_diag"], m["q_constrained"], m["biot_b"],
                                     m["inv_m"], m["k_dr"])


@pytest.mark.parametrize("layout", ["kp", "sell", "sell1", "sell2"])
@pytest.mark.parametrize("n,r", [(16, 0), (16, 1), (64, 1)])
def test_spacetime_operator_and_spmv_bit_identical(oracle, monkeypatch, n, r, layout):
    """Canonical space-time CSR and order-fixed SpMV == SparseMatrix::apply on
    the oracle's canonical CSR (sparse.hpp:30-40), bit for bit, in every device
    layout: the Kronecker-paired layout (default: the m rows of one spatial
    pattern on one thread, one index per run of 8 displacement columns) and the
    SELL layout (PDG_SPMV_FORMAT=sell) in both U-class thread mappings (one row
    per thread, two rows sharing the column and x loads; PDG_SPMV_ROWS)."""
    if layout != "kp":
        monkeypatch.setenv("PDG_SPMV_FORMAT", "sell")
    if layout in ("sell1", "sell2"):
        monkeypatch.setenv("PDG_SPMV_ROWS", layout[-1])
    spec = P.config1(n)
    rp = oracle.RefProblem(spec.to_dict())
    T = oracle.time_constants(r)["T"]
    tau = 0.1 if r == 0 else 0.05
    ops = S.SpatialOperators.assemble(spec)
    blk = S.BlockSolver(ops, T, tau, opt=S.SolveOptions(gmres=S.GmresOptions(restart=10)))
    ro, ri, rv = rp.spacetime_csr(T, tau)
    go, gi, gv = blk.csr()
    assert np.array_equal(ro.astype(np.int64), go)
    assert np.array_equal(ri, gi)
    assert np.array_equal(rv, gv)
    x = P.uniform_vector(P.X_SEED, blk.rows)
    assert np.array_equal(blk.apply(x), oracle.csr_apply(ro, ri, rv, x))


def test_spmv_edge_inputs(oracle):
    """Zero, signed-zero and single-cell inputs: 1x1 mesh, x = 0 -> y = 0 exactly."""
    spec = P.config0()
    spec.nx = spec.ny = 1
    rp = oracle.RefProblem(spec.to_dict())
    T = oracle.time_constants(1)["T"]
    ops = S.SpatialOperators.assemble(spec)
    blk = S.BlockSolver(ops, T, 0.05)
    ro, ri, rv = rp.spacetime_csr(T, 0.05)
    for x in (np.zeros(blk.rows), -np.zeros(blk.rows), P.uniform_vector(7, blk.rows)):
        assert np.array_equal(blk.apply(x), oracle.csr_apply(ro, ri, rv, x))


@pytest.mark.parametrize("n,lam", [(16, 1.0), (16, 2.0), (32, 1.7)])
def test_preconditioner_matches_oracle(oracle, n, lam):
    """One truncated fixed-stress sweep with exact inner solves
    (fixed_stress.hpp:109-139,177-181): GPU block-tridiagonal Cholesky vs the
    oracle's dense LU / banded Cholesky, and bit-identical repeats."""
    spec = P.config1(n)
    rp = oracle.RefProblem(spec.to_dict())
    ops = S.SpatialOperators.assemble(spec)
    tau = 0.05
    blk = S.BlockSolver(ops, np.array([[lam]]), tau)
    rng = np.random.default_rng(11)
    r = rng.standard_normal(blk.rows)
    z = blk.precondition(r)
    z_ref = rp.precondition(lam, tau, r, backend=0)
    z_band = rp.precondition(lam, tau, r, backend=1)
    # two exact CPU solvers already differ by kappa * eps; the GPU solve must sit in that band
    band = np.linalg.norm(z_band - z_ref) / np.linalg.norm(z_ref)
    assert np.linalg.norm(z - z_ref) <= max(1e-10, 10 * band) * np.linalg.norm(z_ref)
    assert np.array_equal(z, blk.precondition(r))
    # linearity (test_coupling.cpp:308-335)
    r2 = rng.standard_normal(blk.rows)
    z2 = blk.precondition(r2)
    zc = blk.precondition(0.3 * r - 1.7 * r2)
    assert np.max(np.abs(zc - (0.3 * z - 1.7 * z2))) <= 1e-12 * np.max(np.abs(zc))


def test_preconditioner_wide_blocks_matches_oracle(oracle):
    """Displacement blocks wider than 74 cells (8 nx > 592 rows) run the sweep
    kernel with 16 rows per CTA and a partial last CTA (nx = 77: 616 = 38.5 x 16);
    checked against the oracle's banded exact solve (fixed_stress.hpp:109-139)."""
    spec = P.config1(77)
    spec.ny = 12
    spec.k_perm_cells = P.lognormal_field(P.K_SEED, spec.nx * spec.ny)
    rp = oracle.RefProblem(spec.to_dict())
    ops = S.SpatialOperators.assemble(spec)
    blk = S.BlockSolver(ops, oracle.time_constants(1)["T"], 0.05)
    rng = np.random.default_rng(17)
    r = rng.standard_normal(blk.rows)
    z = blk.precondition(r)
    T = oracle.time_constants(1)["T"]
    # the oracle preconditions one time component at a time with lambda = T00
    # after the Schur transform; compare component-wise on the block-diagonal part
    nt = blk.rows // 2
    for c in range(2):
        zc = rp.precondition(float(T[0, 0]), 0.05, r[c * nt:(c + 1) * nt], backend=1)
        assert np.linalg.norm(z[c * nt:(c + 1) * nt] - zc) <= 1e-10 * np.linalg.norm(zc)
    assert np.array_equal(z, blk.precondition(r))


@pytest.mark.parametrize("candidate", ["reference", "flexible"])
def test_march_config0_parity(oracle, candidate):
    """BASELINE config 0 (16^2, dG(0), 10 slabs): iterations +-1, per-slab rel L2 <= 1e-9."""
    g = np.load(os.path.join(GOLDEN, "config0_oracle.npz"))
    spec = P.config0()
    run = P.RUNS["config0"]
    ops = S.SpatialOperators.assemble(spec)
    opt = S.SolveOptions(gmres=S.GmresOptions(tol=run["tol"], restart=run["restart"]), candidate=candidate)
    reps, states = S.march(ops, run["r"], run["T"], run["n_slabs"], opt, keep_states=True)
    for s, rep in enumerate(reps):
        assert rep.converged
        assert abs(rep.iterations - int(g["iterations"][s])) <= 1
        ref = g["states"][s].ravel()
        assert np.linalg.norm(states[s] - ref) <= SOLVE_RTOL * np.linalg.norm(ref)


def test_march_terzaghi_reproduces_reference_log():
    """The reference's recorded iteration log (proj/out/iterations.csv) on the GPU:
    identical iteration counts; final residuals to the log's precision band."""
    ref = json.load(open(os.path.join(GOLDEN, "reference_iterations.json")))
    g = np.load(os.path.join(GOLDEN, "terzaghi_oracle.npz"))
    spec = P.terzaghi_recorded()
    run = P.RUNS["terzaghi_recorded"]
    ops = S.SpatialOperators.assemble(spec)
    opt = S.SolveOptions(gmres=S.GmresOptions(tol=run["tol"], restart=run["restart"]))
    reps, states = S.march(ops, run["r"], run["T"], run["n_slabs"], opt, keep_states=True)
    assert [r.iterations for r in reps] == ref["gmres_iterations"]
    np.testing.assert_allclose([r.final_relative_residual for r in reps], ref["final_residual"], rtol=1e-3)
    for s in range(len(reps)):
        refs = g["states"][s].ravel()
        assert np.linalg.norm(states[s] - refs) <= SOLVE_RTOL * np.linalg.norm(refs)


def test_block_solve_upload_path_matches_oracle(oracle):
    """pdg_ops_upload (reference-assembled CSR) + pdg_block_solve == oracle block solve."""
    spec = P.config1(24)
    rp = oracle.RefProblem(spec.to_dict())
    ops = _upload_from_oracle(rp, spec)
    t = oracle.time_constants(1)
    tau = 0.05
    u_prev = np.zeros(rp.n_u)
    p_prev = np.zeros(rp.n_p)
    R = rp.slab_rhs(1, 0.0, tau, u_prev, p_prev)
    shat = rp.schur_forward(1, R)
    x_ref, rep_ref = rp.block_solve(1, tau, shat, tol=1e-10, restart=50, backend=0)
    opt = S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=50))
    blk = S.BlockSolver(ops, t["T"], tau, opt=opt)
    x, rep = blk.solve(shat)
    assert rep.converged and abs(rep.iterations - rep_ref["iterations"]) <= 1
    assert np.linalg.norm(x - x_ref) <= SOLVE_RTOL * np.linalg.norm(x_ref)
    assert len(rep.residual_history) == rep.iterations + 1


def test_nonconvergence_raises_solver_error():
    """max_iter too small -> SolverError with the reference's message (slab.hpp:228-230)."""
    spec = P.config1(16)
    ops = S.SpatialOperators.assemble(spec)
    T = np.array([[1.0]])
    blk = S.BlockSolver(ops, T, 0.1, opt=S.SolveOptions(gmres=S.GmresOptions(tol=1e-14, restart=1, max_iter=1)))
    rhs = P.uniform_vector(5, blk.rows)
    with pytest.raises(S.SolverError, match=r"slab block 0: GMRES did not converge \(rel res"):
        blk.solve(rhs)


def test_zero_rhs_and_invalid_args():
    spec = P.config0()
    ops = S.SpatialOperators.assemble(spec)
    blk = S.BlockSolver(ops, np.array([[1.0]]), 0.1)
    x, rep = blk.solve(np.zeros(blk.rows))
    assert rep.converged and rep.iterations == 0 and not np.any(x)
    with pytest.raises(S.InvalidArgument):
        S.BlockSolver(ops, np.array([[1.0]]), -0.1)
    with pytest.raises(S.InvalidArgument):
        S.BlockSolver(ops, np.array([[1.0]]), 0.1, opt=S.SolveOptions(gmres=S.GmresOptions(tol=2.0)))
    bad = P.config0()
    bad.penalty = -1.0
    with pytest.raises(S.InvalidArgument):
        S.SpatialOperators.assemble(bad)


@pytest.fixture(scope="module")
def config1_oracle_march(oracle):
    """The oracle's full config-1 march (20 slabs, exact sparse-direct inner
    solves, the reference's gmres candidate x + P(V y)), computed once."""
    spec = P.config1(128)
    run = P.RUNS["config1"]
    rp = oracle.RefProblem(spec.to_dict())
    return rp.march(run["r"], run["T"], run["n_slabs"], tol=run["tol"], restart=run["restart"], backend=1,
                    keep_states=True)


@pytest.mark.parametrize("candidate", ["reference", "flexible"])
def test_march_config1_parity(config1_oracle_march, candidate):
    """BASELINE config 1 (128^2, dG(1), lognormal K), all 20 slabs, for both GPU
    GMRES candidates (the headline bench times "flexible"): every slab's
    iteration count within +-1 of the oracle's and its state within relative L2
    1e-9; the final relative residuals both below tol."""
    ref = config1_oracle_march
    spec = P.config1(128)
    run = P.RUNS["config1"]
    ops = S.SpatialOperators.assemble(spec)
    opt = S.SolveOptions(gmres=S.GmresOptions(tol=run["tol"], restart=run["restart"]), candidate=candidate)
    reps, states = S.march(ops, run["r"], run["T"], run["n_slabs"], opt, keep_states=True)
    assert len(reps) == run["n_slabs"] == len(ref["iterations"])
    worst = 0.0
    for s in range(run["n_slabs"]):
        assert reps[s].converged and reps[s].final_relative_residual <= run["tol"]
        assert abs(reps[s].iterations - int(ref["iterations"][s])) <= 1, (s, reps[s].iterations, ref["iterations"])
        assert len(reps[s].residual_history) == reps[s].iterations + 1
        rs = ref["states"][s].ravel()
        d = np.linalg.norm(states[s] - rs) / np.linalg.norm(rs)
        worst = max(worst, d)
        assert d <= SOLVE_RTOL, (s, d)
    print(f"config1 {candidate}: iterations {[r.iterations for r in reps]} "
          f"(oracle {list(ref['iterations'])}), worst per-slab rel L2 {worst:.3e}")


@pytest.mark.parametrize("candidate", ["reference", "flexible"])
def test_gmres_history_is_true_residual(oracle, candidate):
    """SolverReport::residual_history (gmres.hpp:18: true-residual norms, entry 0
    the initial residual) of the GPU solve against the oracle's gmres /
    gmres_flexible on the same dG(1) block (32^2, lognormal K): same length,
    every entry to roundoff. In the flexible path the per-step entries are the
    Arnoldi-relation residual r0 - (A Z) y, equal to b - A (x + Z y) in exact
    arithmetic; the entry that ends the solve is the explicit one."""
    spec = P.config1(32)
    rp = oracle.RefProblem(spec.to_dict())
    ops = S.SpatialOperators.assemble(spec)
    t = oracle.time_constants(1)
    tau = 0.05
    R = rp.slab_rhs(1, 0.0, tau, np.zeros(rp.n_u), np.zeros(rp.n_p))
    shat = rp.schur_forward(1, R)
    # tolerances above the roundoff floor of the reference candidate's true residual (at 1e-12
    # the oracle's x + P(V y) stagnates until the restart, 51 iterations, while x + Z y converges)
    for tol in (1e-8, 1e-10):
        x_ref, rep_ref = rp.block_solve(1, tau, shat, tol=tol, restart=50, backend=1, flexible=candidate == "flexible")
        blk = S.BlockSolver(ops, t["T"], tau, opt=S.SolveOptions(gmres=S.GmresOptions(tol=tol, restart=50),
                                                                 candidate=candidate))
        x, rep = blk.solve(shat)
        h, hr = np.asarray(rep.residual_history), np.asarray(rep_ref["history"])
        assert rep.iterations == rep_ref["iterations"] and len(h) == len(hr) == rep.iterations + 1
        assert h[0] == pytest.approx(hr[0], rel=1e-14)
        assert np.allclose(h, hr, rtol=1e-4, atol=1e-13 * hr[0]), (h, hr)
        assert h[-1] / h[0] <= tol and rep.final_relative_residual == pytest.approx(h[-1] / h[0], rel=1e-14)
        assert np.linalg.norm(x - x_ref) <= SOLVE_RTOL * np.linalg.norm(x_ref)


def _slab_rhs_sequence(rp, r, tau, states):
    nu, nq = rp.n_u, rp.n_q
    u_prev, p_prev = np.zeros(nu), np.zeros(rp.n_p)
    out = []
    for n in range(len(states)):
        out.append(rp.slab_rhs(r, n * tau, tau, u_prev, p_prev))
        end = np.asarray(states[n]).reshape(r + 1, -1)[r]
        u_prev, p_prev = end[:nu], end[nu + nq:]
    return out


@pytest.mark.parametrize("which,r", [("config0", 0), ("config1_16", 1)])
def test_mass_residual_bit_identical(oracle, which, r):
    """pdg_mass_residual == local_mass_residual (slab.hpp:292-318) on the same
    slab systems and states, bit for bit (residual per cell and scale)."""
    spec = P.config0() if which == "config0" else P.config1(16)
    rp = oracle.RefProblem(spec.to_dict())
    ops = S.SpatialOperators.assemble(spec)
    tau = 0.1 if r == 0 else 0.05
    run = rp.march(r, 3 * tau, 3, tol=1e-10, restart=50, keep_states=True)
    rhs = _slab_rhs_sequence(rp, r, tau, run["states"])
    for n in range(3):
        res_ref, sc_ref = rp.mass_residual(r, tau, rhs[n], run["states"][n])
        res, sc = ops.mass_residual(r, tau, rhs[n], run["states"][n])
        assert np.array_equal(res, res_ref) and sc == sc_ref


@pytest.mark.parametrize("r", [0, 1])
def test_march_mass_conservation_terzaghi(r):
    """Acceptance criterion 7 (acceptance.cpp:347-355) on the GPU march: the
    Terzaghi column's per-cell mass residual <= 1e-10 x scale every slab,
    computed on the device (march(..., mass_check=True))."""
    spec = P.terzaghi_recorded()
    spec.ny, spec.lx = 32, 1.0 / 32
    ops = S.SpatialOperators.assemble(spec)
    opt = S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=100))
    reps, _ = S.march(ops, r, 0.1, 5, opt, mass_check=True)
    for rep in reps:
        assert rep.mass_rel is not None and rep.mass_rel <= 1e-10


def test_march_mass_balance_config1(oracle):
    """Config-1 material (lognormal K, dG(1)) on the device: the per-slab mass
    balance of the GPU's GMRES solution (slab.hpp:292-318) matches the oracle's
    on the same problem (32^2), and stays at the same level on the full 128^2
    config (GMRES tol 1e-10 bounds the block residual, not each cell's balance
    against the largest cell scale, so the heterogeneous field sits well above
    1e-10 for both implementations)."""
    opt = S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=50), candidate="flexible")
    spec = P.config1(32)
    rp = oracle.RefProblem(spec.to_dict())
    run = rp.march(1, 0.1, 2, tol=1e-10, restart=50, keep_states=True)
    rhs = _slab_rhs_sequence(rp, 1, 0.05, run["states"])
    ref = [(lambda a: a[0].max() / a[1])(rp.mass_residual(1, 0.05, rhs[n], run["states"][n])) for n in range(2)]
    reps, _ = S.march(S.SpatialOperators.assemble(spec), 1, 0.1, 2, opt, mass_check=True)
    for rep, rr in zip(reps, ref):
        assert rep.mass_rel <= 3.0 * rr + 1e-12, (rep.mass_rel, rr)
    reps, _ = S.march(S.SpatialOperators.assemble(P.config1()), 1, 0.1, 2, opt, mass_check=True)
    for rep in reps:
        assert rep.converged and rep.mass_rel < 1e-7, rep.mass_rel


@pytest.mark.parametrize("r", [0, 1])
def test_slab_rhs_device_bit_identical(oracle, r):
    """pdg_slab_rhs_device == build_slab_system (slab.hpp:58-87) with a nonzero
    jump: R_i = (tau w_i) b(t_i) + phi_i(0) D(u_prev, p_prev), bit for bit."""
    import torch

    spec = P.config1(16)
    rp = oracle.RefProblem(spec.to_dict())
    ops = S.SpatialOperators.assemble(spec)
    tau, t0 = 0.05, 0.35
    slab = S.SlabSolver(ops, r, tau)
    u_prev = P.uniform_vector(3, ops.n_u)
    p_prev = P.uniform_vector(4, ops.n_p)
    dev = torch.device("cuda")
    u = torch.tensor(u_prev, dtype=torch.float64, device=dev)
    p = torch.tensor(p_prev, dtype=torch.float64, device=dev)
    out = torch.empty((r + 1) * ops.n_total, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    slab.rhs_device(t0, u.data_ptr(), p.data_ptr(), out.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), rp.slab_rhs(r, t0, tau, u_prev, p_prev))
    # a slab whose own length differs from the solver's in the last bits (march.hpp:63-72)
    tau2 = 0.30000000000000004 - 0.25
    slab.rhs_device(0.25, u.data_ptr(), p.data_ptr(), out.data_ptr(), tau=tau2)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), rp.slab_rhs(r, 0.25, tau2, u_prev, p_prev))


def test_iteration_log_from_gpu_march():
    """The GPU march's iteration log (csv.hpp:56-71 schema) against the
    reference's recorded proj/out/iterations.csv: identical fields, logged
    residuals to the log's precision band; the driver line format."""
    from paper_1801_04984_b200 import runlog

    ref = json.load(open(os.path.join(GOLDEN, "reference_iterations.json")))
    spec = P.terzaghi_recorded()
    run = P.RUNS["terzaghi_recorded"]
    ops = S.SpatialOperators.assemble(spec)
    opt = S.SolveOptions(gmres=S.GmresOptions(tol=run["tol"], restart=run["restart"]))
    reps, _ = S.march(ops, run["r"], run["T"], run["n_slabs"], opt)
    t_points = S.uniform_partition(run["T"], run["n_slabs"])
    lines = runlog.iteration_log_lines(reps, t_points, run["r"])
    assert lines[0] == ref["lines"][0] and len(lines) == len(ref["lines"])
    for a, b in zip(lines[1:], ref["lines"][1:]):
        fa, fb = a.split(","), b.split(",")
        assert fa[:6] == fb[:6], (a, b)
        assert abs(float(fa[6]) - float(fb[6])) <= 1e-3 * float(fb[6]), (a, b)
    assert runlog.slab_line(9, t_points[10], reps[9], run["r"]).startswith("slab    9  t_n=0.2          method=")


@pytest.mark.parametrize("r", [0, 1])
def test_fixed_stress_march_config0_matches_oracle(oracle, r):
    """Fixed-stress march (march.hpp:80-108, fixed_stress.hpp:144-172) of config
    0 on the device vs the oracle, dG(0) and dG(1) (full Theta = G_hat, Radau
    weights: the coupled flow Schur complement by twisted block LU): identical
    sweep counts per slab and per-slab states within 1e-9 (both converge the
    true residual to 1e-10)."""
    spec = P.config0()
    run = P.RUNS["config0"]
    rp = oracle.RefProblem(spec.to_dict())
    ref = rp.march_fs(r, run["T"], run["n_slabs"], tol=1e-10, max_sweeps=200, keep_states=True)
    ops = S.SpatialOperators.assemble(spec)
    reps, states = S.march(ops, r, run["T"], run["n_slabs"], S.SolveOptions(), keep_states=True,
                           method="fixed-stress")
    for n, rep in enumerate(reps):
        assert rep.converged and rep.iterations == int(ref["sweeps"][n]), (n, rep.iterations, ref["sweeps"][n])
        refs = ref["states"][n].ravel()
        assert np.linalg.norm(states[n] - refs) <= SOLVE_RTOL * np.linalg.norm(refs)


def test_fixed_stress_solver_errors():
    """Argument errors follow FixedStressConfig::validate (fixed_stress.hpp:29-34);
    dG(r >= 2) is refused on the device with a clear message."""
    ops = S.SpatialOperators.assemble(P.config0())
    with pytest.raises(S.InvalidArgument):
        S.FixedStressSolver(ops, 0, 0.1, S.FixedStressConfig(tol=2.0))
    with pytest.raises(S.InvalidArgument):
        S.FixedStressSolver(ops, 2, 0.1)
    fs = S.FixedStressSolver(ops, 0, 0.1, S.FixedStressConfig(max_sweeps=1, tol=1e-15))
    with pytest.raises(S.SolverError, match="fixed-stress did not converge"):
        fs.solve(P.uniform_vector(5, ops.n_total))


@pytest.mark.parametrize("strips", [2, 3])
def test_flow_substructured_strips_match_oracle(oracle, monkeypatch, strips):
    """Opt-in substructured flow solve (PDG_FLOW_STRIPS: strip interiors by
    twisted sweeps, separator system, spike corrections; blocktri_dense.cu):
    the same preconditioner as fixed_stress.hpp:109-139 within the exact-solver
    band, bit-identical repeats; its linear-map roundoff stays below 1e-10."""
    monkeypatch.setenv("PDG_FLOW_STRIPS", str(strips))
    spec = P.config1(32)
    rp = oracle.RefProblem(spec.to_dict())
    ops = S.SpatialOperators.assemble(spec)
    blk = S.BlockSolver(ops, np.array([[1.7]]), 0.05)
    rng = np.random.default_rng(11)
    r = rng.standard_normal(blk.rows)
    z = blk.precondition(r)
    z_ref = rp.precondition(1.7, 0.05, r, backend=0)
    z_band = rp.precondition(1.7, 0.05, r, backend=1)
    band = np.linalg.norm(z_band - z_ref) / np.linalg.norm(z_ref)
    assert np.linalg.norm(z - z_ref) <= max(1e-10, 10 * band) * np.linalg.norm(z_ref)
    assert np.array_equal(z, blk.precondition(r))
    r2 = rng.standard_normal(blk.rows)
    zc = blk.precondition(0.3 * r - 1.7 * r2)
    assert np.max(np.abs(zc - (0.3 * z - 1.7 * blk.precondition(r2)))) <= 1e-10 * np.max(np.abs(zc))


@pytest.mark.parametrize("world", [2, 3])
def test_strip_spmv_is_the_single_gpu_spmv(oracle, world):
    """Multi-GPU row partitioning on one device, rank by rank (no inter-rank
    waits): each strip's SpMV, fed only its owned entries plus the exchange set
    (parallel.strip_exchange_sets), reproduces its rows of the single-GPU
    order-fixed SpMV bit for bit, and the strips cover every row once."""
    import torch

    from paper_1801_04984_b200 import parallel as par

    n, m = 32, 2
    ops = S.SpatialOperators.assemble(P.config1(n))
    op = S.SpaceTimeOperator(ops, oracle.time_constants(1)["T"], 0.05)
    x = torch.from_numpy(P.uniform_vector(P.X_SEED, op.rows)).cuda()
    y_ref = torch.empty_like(x)
    op.apply_device(x.data_ptr(), y_ref.data_ptr())
    strips = par.strip_partition(n, world)
    owner = par.row_owner(n, n, m, strips)
    covered = np.zeros(op.rows, dtype=bool)
    for k in range(world):
        sp = par.DeviceStripSpMV(op, n, n, m, k, world, dist=None)
        _, recv = par.strip_exchange_sets(n, n, m, strips, k)
        keep = owner == k
        for v in recv.values():
            keep[v] = True
        xk = x.clone()
        xk[torch.from_numpy(~keep).cuda()] = float("nan")  # anything outside owned + halo must not be read
        yk = torch.full_like(x, float("nan"))
        sp.apply(xk, yk)
        own = torch.from_numpy(owner == k).cuda()
        assert torch.equal(yk[own], y_ref[own]), k
        covered |= owner == k
    assert covered.all()


@pytest.mark.parametrize("restart,candidate", [(2, "reference"), (3, "flexible"), (1, "reference")])
def test_gmres_restart_accounting_matches_oracle(oracle, restart, candidate):
    """Restarted GMRES (gmres.hpp:75-131: m = min(restart, left), true residual
    recomputed at each cycle start, history of true residuals): with a restart
    far below the iteration count, the GPU walks the same cycles as the oracle:
    same iteration count, same residual history to roundoff, same solution."""
    spec = P.config1(16)
    rp = oracle.RefProblem(spec.to_dict())
    ops = S.SpatialOperators.assemble(spec)
    t = oracle.time_constants(1)
    tau = 0.05
    R = rp.slab_rhs(1, 0.0, tau, np.zeros(rp.n_u), np.zeros(rp.n_p))
    shat = rp.schur_forward(1, R)
    x_ref, rep_ref = rp.block_solve(1, tau, shat, tol=1e-10, restart=restart, max_iter=400, backend=0,
                                    flexible=candidate == "flexible")
    blk = S.BlockSolver(ops, t["T"], tau, opt=S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=restart),
                                                             candidate=candidate))
    x, rep = blk.solve(shat)
    assert rep.converged and rep_ref["converged"]
    assert abs(rep.iterations - rep_ref["iterations"]) <= 1, (rep.iterations, rep_ref["iterations"])
    h, hr = np.asarray(rep.residual_history), np.asarray(rep_ref["history"])
    k = min(len(h), len(hr))
    assert np.allclose(h[:k], hr[:k], rtol=1e-6, atol=1e-9 * hr[0])
    assert np.linalg.norm(x - x_ref) <= SOLVE_RTOL * np.linalg.norm(x_ref)


def test_march_nonsquare_mixed_bcs_matches_oracle(oracle):
    """A non-square mesh (nx != ny), non-unit domain and every boundary kind
    (fixed / roller_x / roller_y / traction; pressure / no_flow) through the
    whole device march (dG(1), 3 slabs) vs the oracle: iterations +-1, states
    within 1e-9."""
    spec = P.config1(6)
    spec.nx, spec.ny = 12, 7
    spec.k_perm_cells = P.lognormal_field(P.K_SEED, spec.nx * spec.ny)
    spec.disp = {"left": ("fixed", (0.0, 0.0)), "right": ("roller_x", (0.0, 0.3)),
                 "bottom": ("roller_y", (0.2, 0.0)), "top": ("traction", (0.1, -1.0))}
    spec.flow = {"left": ("pressure", 0.5), "right": ("no_flow", 0.0), "bottom": ("no_flow", 0.0),
                 "top": ("pressure", -0.25)}
    spec.lx, spec.ly = 1.3, 0.9
    rp = oracle.RefProblem(spec.to_dict())
    ref = rp.march(1, 0.15, 3, tol=1e-10, restart=50, keep_states=True, backend=0)
    ops = S.SpatialOperators.assemble(spec)
    reps, states = S.march(ops, 1, 0.15, 3, S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=50)),
                           keep_states=True)
    for n, rep in enumerate(reps):
        assert rep.converged and abs(rep.iterations - int(ref["iterations"][n])) <= 1
        refs = ref["states"][n].ravel()
        assert np.linalg.norm(states[n] - refs) <= SOLVE_RTOL * np.linalg.norm(refs)


@pytest.mark.parametrize("nb,m", [(9, 40), (16, 33), (2, 17), (1, 24)])
def test_block_tridiagonal_lu_sweep(nb, m):
    """Non-symmetric block-tridiagonal solve (twisted block LU with in-block
    partial pivoting, the same dense sweep kernel): against a dense solve, for
    one and two right-hand sides, including 1- and 2-block chains."""
    import scipy.sparse as sp
    import torch

    from paper_1801_04984_b200 import distributed as D

    rng = np.random.default_rng(nb * 100 + m)
    n = nb * m
    A = np.zeros((n, n))
    for j in range(nb):
        s = slice(j * m, (j + 1) * m)
        A[s, s] = rng.standard_normal((m, m)) + 4 * m * np.eye(m) * (1 + rng.random())
        if j + 1 < nb:
            t = slice((j + 1) * m, (j + 2) * m)
            A[t, s] = rng.standard_normal((m, m))
            A[s, t] = rng.standard_normal((m, m)) * 0.5
    solver = D.TriSolver(sp.csr_matrix(A), [m] * nb, symmetric=False)
    B = rng.standard_normal((n, 2))
    x = solver.solve(torch.as_tensor(B, device="cuda")).cpu().numpy()
    ref = np.linalg.solve(A, B)
    assert np.linalg.norm(x - ref) <= 1e-12 * np.linalg.norm(ref)
    x1 = solver.solve(torch.as_tensor(B[:, 0], device="cuda")).cpu().numpy()
    assert np.linalg.norm(x1 - ref[:, 0]) <= 1e-12 * np.linalg.norm(ref[:, 0])


@pytest.mark.parametrize("solver", ["local", "general"])
def test_nested_dissection_inner_solves_match_block_tridiagonal(monkeypatch, solver):
    """The nested-dissection multifrontal inner solves (csrc/nd.cu, the default)
    and the twisted block-tridiagonal ones (PDG_A_SOLVER=local|general,
    PDG_FLOW_SOLVER=blocktri) are both exact: the preconditioner outputs agree to
    roundoff, and ND repeats are bit-identical (fixed-order dataflow)."""
    spec = P.config1(32)
    ops = S.SpatialOperators.assemble(spec)
    rng = np.random.default_rng(5)
    theta = np.array([[1.7]])
    blk = S.BlockSolver(ops, theta, 0.05)
    r = rng.standard_normal(blk.rows)
    z_nd = blk.precondition(r)
    assert np.array_equal(z_nd, blk.precondition(r))
    monkeypatch.setenv("PDG_A_SOLVER", solver)
    monkeypatch.setenv("PDG_FLOW_SOLVER", "blocktri")
    blk2 = S.BlockSolver(ops, theta, 0.05)
    z_bt = blk2.precondition(r)
    # both exact; they differ by roundoff amplified by the conditioning of A and S_q
    # (lognormal permeability): ~2e-11 relative measured
    assert np.linalg.norm(z_nd - z_bt) <= 1e-9 * np.linalg.norm(z_bt)


@pytest.mark.parametrize("candidate,restart", [("flexible", 50), ("reference", 50), ("flexible", 2)])
def test_gmres_loop_variants_agree(monkeypatch, candidate, restart):
    """The GMRES loop variants on one dG(1) block (16^2, lognormal K):
    - default, flexible: device-driven steps (the Gram-Schmidt kernel applies the
      Givens rotations and decides the stop from || beta e1 - H y ||; the next step is
      queued before the host reads the stop flag, and skipped on the device);
    - PDG_GMRES_HOST_LOOP=1: the host-driven loop (Arnoldi-relation residual
      r0 - (A Z) y each step), the reference candidate's loop;
    - PDG_SPMV_DOTS=0: the first Gram-Schmidt pass as its own multidot instead of
      the SpMV epilogue; PDG_KRYLOV_UNFUSED=1: the launch-per-step sequence.
    The fused cooperative kernels keep the partial-sum order of the launch-per-step
    sequence (bit-identical once the SpMV dots are off); every variant is
    deterministic and takes the same iterations, solutions within 1e-10.
    restart=2 exercises cycle ends without convergence."""
    spec = P.config1(16)
    ops = S.SpatialOperators.assemble(spec)
    t = S.time_constants(1)
    rhs = np.random.default_rng(11).standard_normal(2 * ops.n_total)
    opt = S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=restart), candidate=candidate)
    blk = S.BlockSolver(ops, t["T"], 0.05, opt=opt)
    x_f, rep_f = blk.solve(rhs)
    x_r, rep_r = blk.solve(rhs)
    assert rep_f.converged and np.array_equal(x_f, x_r)
    assert np.array_equal(np.asarray(rep_f.residual_history), np.asarray(rep_r.residual_history))
    runs = []
    for env in ({"PDG_GMRES_HOST_LOOP": "1"}, {"PDG_GMRES_HOST_LOOP": "1", "PDG_SPMV_DOTS": "0"},
                {"PDG_GMRES_HOST_LOOP": "1", "PDG_SPMV_DOTS": "0", "PDG_KRYLOV_UNFUSED": "1"}):
        for k in ("PDG_GMRES_HOST_LOOP", "PDG_SPMV_DOTS", "PDG_KRYLOV_UNFUSED"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        runs.append(blk.solve(rhs))
    (x_s, rep_s), (x_u, rep_u) = runs[1], runs[2]
    assert rep_s.iterations == rep_u.iterations and np.array_equal(x_s, x_u)
    assert np.array_equal(np.asarray(rep_s.residual_history), np.asarray(rep_u.residual_history))
    for x_v, rep_v in runs:
        assert rep_v.converged and rep_v.iterations == rep_f.iterations, (rep_v.iterations, rep_f.iterations)
        assert len(rep_v.residual_history) == len(rep_f.residual_history) == rep_f.iterations + 1
        assert np.linalg.norm(x_v - x_f) <= 1e-10 * np.linalg.norm(x_f)
        h, hv = np.asarray(rep_f.residual_history), np.asarray(rep_v.residual_history)
        assert np.allclose(h, hv, rtol=1e-6, atol=1e-12 * h[0])


def test_spmv_config3_256_bit_identical(oracle):
    """BASELINE config 3 at 256^2 (dG(1), 1.44M rows, 59.6M nnz): the device-built
    canonical CSR and y = A x (x ~ U(-1,1), seed 4984) equal the oracle's CSR and
    SparseMatrix::apply on it bit for bit (the two-row thread mapping runs here)."""
    spec = P.config3(256)
    T = oracle.time_constants(1)["T"]
    op = S.SpaceTimeOperator(S.SpatialOperators.assemble(spec), T, 0.05)
    assert op.rows == 1442816 and op.nnz == 59583488
    go, gi, gv = op.csr()
    rp = oracle.RefProblem(spec.to_dict())
    ro, ri, rv = rp.spacetime_csr(T, 0.05)
    assert np.array_equal(ro.astype(np.int64), go)
    assert np.array_equal(ri, gi)
    assert np.array_equal(rv, gv)
    del gi, gv
    import torch
    x = P.uniform_vector(P.X_SEED, op.rows)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    op.apply_device(xd.data_ptr(), yd.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(yd.cpu().numpy(), oracle.csr_apply(ro, ri, rv, x))


def test_spmv_config3_512_bit_identical(oracle):
    """BASELINE config 3 at 512^2 (5.77M rows, 238.7M nnz): the device-built
    canonical CSR equals the oracle-built one, and y = A x equals the oracle's
    SparseMatrix::apply (sparse.hpp:30-40) on it, bit for bit."""
    import torch
    spec = P.config3(512)
    T = oracle.time_constants(1)["T"]
    op = S.SpaceTimeOperator(S.SpatialOperators.assemble(spec), T, 0.05)
    assert op.rows == 5769216 and op.nnz == 238704640
    x = P.uniform_vector(P.X_SEED, op.rows)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    op.apply_device(xd.data_ptr(), yd.data_ptr())
    torch.cuda.synchronize()
    y = yd.cpu().numpy()
    del xd, yd
    go, gi, gv = op.csr()
    del op
    rp = oracle.RefProblem(spec.to_dict())
    ro, ri, rv = rp.spacetime_csr(T, 0.05)
    del rp
    assert np.array_equal(ro.astype(np.int64), go)
    assert np.array_equal(ri, gi)
    assert np.array_equal(rv, gv)
    del gi, gv
    assert np.array_equal(y, oracle.csr_apply(ro, ri, rv, x, threads=os.cpu_count()))


def test_spmv_config3_1024_bit_identical_to_cpu(oracle):
    """BASELINE config 3 at 1024^2 (23.1M rows, 955.6M nnz): y = A x on the GPU
    equals the oracle's SparseMatrix::apply (sparse.hpp:30-40, sequential row
    sums, no FMA) over the same canonical CSR, downloaded from the device (the
    device CSR equals the oracle-built one at 16^2..512^2), bit for bit; the
    row structure matches the closed form of SURVEY Appendix B."""
    import torch
    psutil = pytest.importorskip("psutil")
    if psutil.virtual_memory().available < 40e9:
        pytest.skip("needs ~40 GB of host memory for the 12 GB CSR and the checks")
    T = S.time_constants(1)["T"]
    op = S.SpaceTimeOperator(S.SpatialOperators.assemble(P.config3(1024)), T, 0.05)
    assert op.rows == 23072768 and op.nnz == 955559936
    x = P.uniform_vector(P.X_SEED, op.rows)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    op.apply_device(xd.data_ptr(), yd.data_ptr())
    torch.cuda.synchronize()
    y = yd.cpu().numpy()
    off, idx, val = op.csr()
    assert off[0] == 0 and off[-1] == op.nnz and np.all(np.diff(off) > 0)
    yc = oracle.csr_apply(off, idx, val, x, threads=os.cpu_count())
    assert np.array_equal(y, yc)


def test_spmv_config3_1024_properties(monkeypatch):
    """BASELINE config 3 at full size (1024^2, 23.1M rows, 955.6M nnz), through
    size-independent properties: the Kronecker-paired layout and both SELL-layout
    U-class thread mappings give the same bits, repeated applications are
    bit-identical, A (2 x) = 2 A x exactly (a power-of-two scaling commutes with
    every rounding), and A 0 = 0."""
    import torch
    T = S.time_constants(1)["T"]
    ops = S.SpatialOperators.assemble(P.config3(1024))
    op = S.SpaceTimeOperator(ops, T, 0.05)
    assert op.rows == 23072768 and op.nnz == 955559936
    x = torch.from_numpy(P.uniform_vector(P.X_SEED, op.rows)).cuda()
    y1, y2, y3 = (torch.empty_like(x) for _ in range(3))
    op.apply_device(x.data_ptr(), y1.data_ptr())
    op.apply_device(x.data_ptr(), y2.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    monkeypatch.setenv("PDG_SPMV_FORMAT", "sell")
    op_sell = S.SpaceTimeOperator(ops, T, 0.05)
    assert op_sell.nnz == op.nnz
    for rows in ("1", "2"):
        monkeypatch.setenv("PDG_SPMV_ROWS", rows)
        y3.fill_(1.0)
        torch.cuda.synchronize()  # torch's stream and the library's do not order each other
        op_sell.apply_device(x.data_ptr(), y3.data_ptr())
        torch.cuda.synchronize()
        assert torch.equal(y1, y3)
    del op_sell
    monkeypatch.delenv("PDG_SPMV_ROWS")
    monkeypatch.delenv("PDG_SPMV_FORMAT")
    x2 = 2.0 * x
    torch.cuda.synchronize()
    op.apply_device(x2.data_ptr(), y2.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(y2, 2.0 * y1)
    x.zero_()
    torch.cuda.synchronize()
    op.apply_device(x.data_ptr(), y2.data_ptr())
    torch.cuda.synchronize()
    assert not torch.any(y2 != 0)


def test_nd_level_kernels_match_chunk_kernel(monkeypatch):
    """The level-synchronous nested-dissection solve (PDG_ND_LEVELS=1; the automatic
    fallback when the chunk kernel's ring / arena do not fit wide fronts) against the
    default chunk kernel: the same exact solves to roundoff, repeats bit-identical."""
    spec = P.config1(32)
    ops = S.SpatialOperators.assemble(spec)
    r = np.random.default_rng(9).standard_normal(2 * ops.n_total)
    T = S.time_constants(1)["T"]
    z_chunk = S.BlockSolver(ops, T, 0.05).precondition(r)
    monkeypatch.setenv("PDG_ND_LEVELS", "1")
    blk = S.BlockSolver(ops, T, 0.05)
    z_lvl = blk.precondition(r)
    assert np.array_equal(z_lvl, blk.precondition(r))
    assert np.linalg.norm(z_lvl - z_chunk) <= 1e-10 * np.linalg.norm(z_chunk)


@pytest.mark.parametrize("n", [192, 256])
def test_large_mesh_slab_solve(n):
    """Meshes whose top separator fronts are too wide for the chunk kernel (the level
    kernels take over): the dG(1) march converges in the config-1 iteration counts
    with the local mass balance of the 128^2 runs."""
    ops = S.SpatialOperators.assemble(P.config3(n))
    opt = S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=50), candidate="flexible")
    reps, _ = S.march(ops, 1, 0.1, 2, opt, mass_check=True)
    for rep in reps:
        assert rep.converged and 3 <= rep.iterations <= 6
        assert rep.mass_rel < 1e-7


# ---- dG(r), r >= 2: several Schur blocks (slab.hpp:194-203, schur.hpp:101-173) ----
@pytest.mark.parametrize("r", [2, 3, 4, 5])
def test_time_constants_high_order(oracle, r):
    """pdg_time_constants for r >= 2 (Hessenberg + Francis QR in the library where the reference
    calls Eigen::RealSchur; the oracle takes LAPACK's): the basis constants agree to roundoff, the
    ordered block structure is the same, Q is orthogonal, Q T Q^T = W, and the diagonal blocks
    carry the same eigenvalues in the same standardized form. (T's off-block entries and Q are
    unique only up to rotations of the invariant subspaces.)"""
    lib, ref = S.time_constants(r), oracle.time_constants(r)
    n = r + 1
    for k in ("nodes", "weights", "phi_at0", "G_hat"):
        assert np.allclose(lib[k], ref[k], rtol=1e-13, atol=1e-14), k
    sizes, starts = oracle.schur_blocks(r)
    assert np.array_equal(lib["block_sizes"], sizes) and np.array_equal(lib["block_starts"], starts)
    W = lib["G_hat"] / lib["weights"][:, None]
    T, Q = lib["T"], lib["Q"]
    assert abs(Q.T @ Q - np.eye(n)).max() <= 1e-12
    assert abs(Q @ T @ Q.T - W).max() <= 1e-10 * (1 + abs(W).max())
    for s, i in zip(sizes, starts):
        assert np.allclose(np.diag(T)[i:i + s], np.diag(ref["T"])[i:i + s], rtol=1e-11)
        if s == 2:
            assert T[i, i] == pytest.approx(T[i + 1, i + 1], rel=1e-13)
            assert T[i, i + 1] * T[i + 1, i] == pytest.approx(ref["T"][i, i + 1] * ref["T"][i + 1, i], rel=1e-10)
            assert (T[i + 2:, i:i + 2] == 0.0).all()
        else:
            assert (T[i + 1:, i] == 0.0).all()


@pytest.mark.parametrize("candidate", ["reference", "flexible"])
@pytest.mark.parametrize("r", [2, 3])
def test_march_high_order_parity(oracle, r, candidate):
    """dG(2) / dG(3) march of a config-0-type problem: one GMRES solve per Schur block in descending
    order with the T_ij D y_j couplings on the device (slab.hpp:194-235). Per slab: the maximum
    block iteration count within +-1 of the oracle's and the state within 1e-9."""
    spec = P.config0()
    rp = oracle.RefProblem(spec.to_dict())
    n_slabs = 3
    ref = rp.march(r, 0.3, n_slabs, tol=1e-10, restart=50, backend=0, flexible=candidate == "flexible",
                   keep_states=True)
    ops = S.SpatialOperators.assemble(spec)
    opt = S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=50), candidate=candidate)
    reps, states = S.march(ops, r, 0.3, n_slabs, opt, keep_states=True, mass_check=True)
    for s in range(n_slabs):
        assert reps[s].converged
        assert abs(reps[s].iterations - int(ref["iterations"][s])) <= 1, (s, reps[s].iterations, ref["iterations"])
        d = np.linalg.norm(states[s] - ref["states"][s].ravel()) / np.linalg.norm(ref["states"][s])
        assert d <= SOLVE_RTOL, (s, d)
        assert reps[s].mass_rel <= 1e-7
    slab = S.SlabSolver(ops, r, 0.1, opt)
    rhs = rp.slab_rhs(r, 0.0, 0.1, np.zeros(rp.n_u), np.zeros(rp.n_p))
    x, rep = slab.solve(rhs)
    blocks = slab.block_reports()
    sizes, _ = oracle.schur_blocks(r)
    assert [b[0] for b in blocks] == list(sizes)
    assert rep.iterations == max(b[1] for b in blocks) and all(b[2] <= 1e-10 for b in blocks)
    assert np.linalg.norm(x - ref["states"][0].ravel()) <= SOLVE_RTOL * np.linalg.norm(ref["states"][0])
    with pytest.raises(S.InvalidArgument):
        S.SlabSolver(ops, 6, 0.1, opt)


# ---- assemble_rhs in full: VolumeData and time-/space-dependent boundary functions ----
def _rhs_variants():
    a = P.config0()
    a.nx, a.ny = 5, 3
    b = P.config1(6)
    b.disp = {"left": ("fixed", (0.0, 0.0)), "right": ("roller_x", (0.0, 0.0)),
              "bottom": ("roller_y", (0.0, 0.0)), "top": ("traction", (0.0, 0.0))}
    b.flow = {"left": ("pressure", 0.0), "right": ("no_flow", 0.0), "bottom": ("no_flow", 0.0), "top": ("pressure", 0.0)}
    b.lx, b.ly = 1.3, 0.9
    c = P.config0()
    c.nx, c.ny = 1, 1
    return [a, b, c]


@pytest.mark.parametrize("spec", _rhs_variants(), ids=lambda s: f"{s.nx}x{s.ny}")
def test_rhs_sampled_bit_identical(oracle, spec):
    """pdg_ops_rhs_sampled == assemble_rhs (assembly.hpp:467-563) with momentum / Darcy / mass
    sources and time- and space-dependent traction, Dirichlet, pressure and prescribed-flux data
    (the eliminated couplings mq_bc / b_bc included), bit for bit: the fields are sampled at the
    quadrature points by the host (here the oracle) and accumulated on the device in the
    reference's order. Sample points as the library documents them; absent fields skipped."""
    rp = oracle.RefProblem(spec.to_dict())
    ops = S.SpatialOperators.assemble(spec)
    rp.set_test_fields(1)
    for t in (0.0, 0.37):
        sm = rp.sample_rhs_data(t)
        u, q, p = rp.assemble_rhs(t)
        gu, gq, gp = ops.rhs_sampled(sm)
        assert np.array_equal(u, gu) and np.array_equal(q, gq) and np.array_equal(p, gp)
        assert np.abs(q).max() > 0 and np.abs(p).max() > 0
    # the documented sample points are the ones the reference evaluates at
    cxy, ids, fxy = ops.sample_points()
    hx, hy = spec.lx / spec.nx, spec.ly / spec.ny
    g6 = oracle.gauss_points(6)
    assert np.array_equal(cxy[0, :, 0].reshape(6, 6)[:, 0], 0 * hx + g6 * hx)
    assert np.array_equal(cxy[-1, :, 1].reshape(6, 6)[0, :], (spec.ny - 1) * hy + g6 * hy)
    assert len(ids) == 2 * (spec.nx + spec.ny) and (np.diff(ids) > 0).all()
    # boundary data only (no volume fields): the volume loops are skipped as in the reference
    rp.set_test_fields(1)
    sm = rp.sample_rhs_data(0.2)
    sm0 = dict(sm, momentum=None, darcy=None, mass=None)
    zero = {k: np.zeros_like(v) for k, v in sm.items()}
    gu0, gq0, gp0 = ops.rhs_sampled(dict(sm0))
    gu1, gq1, gp1 = ops.rhs_sampled(dict(zero, traction=sm["traction"], dirichlet=sm["dirichlet"], flow=sm["flow"]))
    assert np.array_equal(gu0, gu1) and np.array_equal(gq0, gq1) and np.array_equal(gp0, gp1)
    # constant data through the sampled path == the constant-data kernels == the oracle
    rp2 = oracle.RefProblem(spec.to_dict())
    sm = rp2.sample_rhs_data(0.0)
    assert sm["momentum"] is None and sm["darcy"] is None and sm["mass"] is None
    cu, cq, cp = ops.rhs(0.0)
    su, sq, sp_ = ops.rhs_sampled(sm)
    ru, rq, rpp = rp2.assemble_rhs(0.0)
    for a_, b_, c_ in ((ru, cu, su), (rq, cq, sq), (rpp, cp, sp_)):
        assert np.array_equal(a_, b_) and np.array_equal(a_, c_)


def test_march_with_sampled_data(oracle):
    """A dG(1) slab built from sampled, time-dependent data on the device
    (pdg_slab_rhs_sampled_device) equals the oracle's build_slab_system bit for bit, and its
    solve matches the oracle's."""
    import torch
    spec = _rhs_variants()[1]
    rp = oracle.RefProblem(spec.to_dict())
    rp.set_test_fields(1)
    ops = S.SpatialOperators.assemble(spec)
    r, tau, t0 = 1, 0.05, 0.1
    opt = S.SolveOptions(gmres=S.GmresOptions(tol=1e-10, restart=50))
    slab = S.SlabSolver(ops, r, tau, opt)
    nodes = S.time_constants(r)["nodes"]
    u_prev = 0.01 * P.uniform_vector(3, ops.n_u)
    p_prev = 0.01 * P.uniform_vector(4, ops.n_p)
    ref_rhs = rp.slab_rhs(r, t0, tau, u_prev, p_prev)
    samples = [rp.sample_rhs_data(t0 + c * tau) for c in nodes]
    ud, pd = torch.from_numpy(u_prev).cuda(), torch.from_numpy(p_prev).cuda()
    rhs = torch.empty((r + 1) * ops.n_total, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    slab.rhs_sampled_device(samples, ud.data_ptr(), pd.data_ptr(), rhs.data_ptr())
    assert np.array_equal(rhs.cpu().numpy(), ref_rhs)
    x, rep = slab.solve(ref_rhs)
    T = oracle.time_constants(r)
    xr, rr = rp.block_solve(r, tau, rp.schur_forward(r, ref_rhs), tol=1e-10, restart=50, backend=1)
    y = (T["Q"] @ xr.reshape(r + 1, -1)).ravel()
    assert abs(rep.iterations - rr["iterations"]) <= 1
    assert np.linalg.norm(x - y) <= SOLVE_RTOL * np.linalg.norm(y)


def test_mms_poroelastic_march_2d_on_device():
    """The reference's MMS-type use of assemble_rhs (volume sources and space- / time-dependent
    boundary functions, assembly.hpp:467-563) end to end on the GPU in 2D: u = U(x)(1 + t),
    p = P(x)(1 + t/2), q = -(K/eta) grad p, f = -div(sigma(u) - b p I), g = d/dt(b div u + p/M) +
    div q, Nitsche displacement data on left / bottom, traction data on right / top, pressure data
    on left / top and prescribed normal flux on right / bottom; dG(1) (exact in time for this
    solution), two slabs. Nodal displacement error second order, cell pressure at least first order
    under n = 4, 8, 16."""
    import sympy as sy
    import torch
    x, y, t = sy.symbols("x y t")
    lam, mu, bb, MM, eta, kperm = 2.0, 1.5, 0.8, 10.0, 1.0, 1.0
    U = sy.Matrix([sy.sin(sy.pi * x / 2) * sy.cos(y), x * y + sy.sin(x) * y * y]) * sy.Rational(1, 10)
    P_ = sy.sin(sy.pi * x / 2) * sy.cos(y) + x * y
    u = U * (1 + t)
    p = P_ * (1 + t / 2)
    grad = u.jacobian([x, y])
    eps = (grad + grad.T) / 2
    sig_e = 2 * mu * eps + lam * eps.trace() * sy.eye(2)
    sig = sig_e - bb * p * sy.eye(2)
    fm = -sy.Matrix([sum(sy.diff(sig[i, j], (x, y)[j]) for j in range(2)) for i in range(2)])
    q = -(kperm / eta) * sy.Matrix([sy.diff(p, v) for v in (x, y)])
    g = sy.diff(bb * eps.trace() + p / MM, t) + sum(sy.diff(q[i], (x, y)[i]) for i in range(2))
    L = lambda e: sy.lambdify((x, y, t), e, "numpy")  # noqa: E731
    u_f, p_f, fm_f, g_f, q_f, sg_f = L(u), L(p), L(fm), L(g), L(q), L(sig)

    def vec(fn, X, Y, tt):
        out = fn(X, Y, tt)
        return np.stack([np.broadcast_to(np.asarray(out[i][0], float), X.shape) for i in range(2)], axis=-1)

    def sca(fn, X, Y, tt):
        return np.broadcast_to(np.asarray(fn(X, Y, tt), float), X.shape).copy()

    r, n_slabs, T = 1, 2, 0.5
    tau = T / n_slabs
    nodes = S.time_constants(r)["nodes"]
    opt = S.SolveOptions(gmres=S.GmresOptions(tol=1e-12, restart=50), candidate="flexible")
    normals = {"left": (-1.0, 0.0), "right": (1.0, 0.0), "bottom": (0.0, -1.0), "top": (0.0, 1.0)}
    eu, ep = [], []
    for n in (4, 8, 16):
        spec = P.config0()
        spec.nx = spec.ny = n
        spec.lam, spec.mu, spec.biot_b, spec.biot_m, spec.eta, spec.k_perm = lam, mu, bb, MM, eta, kperm
        spec.disp = {"left": ("fixed", (0.0, 0.0)), "bottom": ("fixed", (0.0, 0.0)),
                     "right": ("traction", (0.0, 0.0)), "top": ("traction", (0.0, 0.0))}
        spec.flow = {"left": ("pressure", 0.0), "top": ("pressure", 0.0), "right": ("no_flow", 0.0),
                     "bottom": ("no_flow", 0.0)}
        ops = S.SpatialOperators.assemble(spec)
        cxy, ids, fxy = ops.sample_points()
        nh = n * (n + 1)
        tags = ["bottom" if f < n else "top" if f < nh else "left" if f < nh + n else "right" for f in ids]
        h = 1.0 / n
        nod = np.array([[((i + (a & 1)) * h, (j + (a >> 1)) * h) for a in range(4)] for j in range(n) for i in range(n)])
        cc = np.array([((i + .5) * h, (j + .5) * h) for j in range(n) for i in range(n)])
        u_prev = torch.from_numpy(vec(u_f, nod[..., 0], nod[..., 1], 0.0).reshape(-1).copy()).cuda()
        p_prev = torch.from_numpy(sca(p_f, cc[:, 0], cc[:, 1], 0.0)).cuda()
        slab = S.SlabSolver(ops, r, tau, opt)
        nt = ops.n_total
        rhs = torch.empty((r + 1) * nt, dtype=torch.float64, device="cuda")
        out = torch.empty_like(rhs)
        for s_ in range(n_slabs):
            samples = []
            for c in nodes:
                tt = s_ * tau + c * tau
                X, Y = fxy[..., 0], fxy[..., 1]
                SG, Q = sg_f(X, Y, tt), q_f(X, Y, tt)
                trac, flow = np.zeros(fxy.shape), sca(p_f, X, Y, tt)
                for b_, tg in enumerate(tags):
                    nv = normals[tg]
                    for i in range(2):
                        trac[b_, :, i] = sum(np.broadcast_to(np.asarray(SG[i][j], float), X.shape)[b_] * nv[j] for j in range(2))
                    if tg in ("right", "bottom"):
                        flow[b_] = sum(np.broadcast_to(np.asarray(Q[j][0], float), X.shape)[b_] * nv[j] for j in range(2))
                samples.append(dict(momentum=vec(fm_f, cxy[..., 0], cxy[..., 1], tt), mass=sca(g_f, cxy[..., 0], cxy[..., 1], tt),
                                    traction=trac, dirichlet=vec(u_f, X, Y, tt), flow=flow))
            torch.cuda.synchronize()
            slab.rhs_sampled_device(samples, u_prev.data_ptr(), p_prev.data_ptr(), rhs.data_ptr())
            rep = slab.solve_device(rhs.data_ptr(), out.data_ptr())
            assert rep.converged
            end = out[r * nt:(r + 1) * nt]
            u_prev.copy_(end[:ops.n_u])
            p_prev.copy_(end[ops.n_u + ops.n_q:])
            torch.cuda.synchronize()
        eu.append(float(np.sqrt(np.mean((u_prev.cpu().numpy() - vec(u_f, nod[..., 0], nod[..., 1], T).reshape(-1)) ** 2))))
        ep.append(float(np.sqrt(np.mean((p_prev.cpu().numpy() - sca(p_f, cc[:, 0], cc[:, 1], T)) ** 2))))
    ru = [np.log2(eu[i] / eu[i + 1]) for i in range(2)]
    rp_ = [np.log2(ep[i] / ep[i + 1]) for i in range(2)]
    print("MMS 2D march: u errors", eu, "rates", ru, "p errors", ep, "rates", rp_)
    assert eu[2] < eu[1] < eu[0] and ep[2] < ep[1] < ep[0]
    assert ru[1] > 1.7 and rp_[1] > 0.9, (eu, ru, ep, rp_)
