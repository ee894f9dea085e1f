"""Pins of the oracle's RHS f(Q, t).

* free-stream preservation (BASELINE.json north_star)
* discrete conservation on periodic meshes; mass and energy on all-wall boxes
* rotation covariance (catches the garbled Eq. 1 and the printed form of Eq. 4)
* brute force: the paper's weak form eq:dgma with the interpolated
  flux, integrated by an independent collapsed Gauss rule on 1-2 elements
* h-convergence at rate N+1 on the exact density/entropy wave (textbook exact
  Euler solution) and on a small-amplitude acoustic pulse vs 3D linear acoustics
"""
import math

import numpy as np
import pytest

import quad
from oracle import euler, timestep
from oracle.rhs import BlowUp, OracleMesh, rhs
from synth import configs
from synth import mesh as smesh

G = 1.4
REST = (1.4, 0.0, 0.0, 0.0, 2.5)


def om(m, N, **kw):
    return OracleMesh(order=N, vxyz=m.vxyz, etov=m.etov, bc=m.bc, etoe=m.etoe, etof=m.etof, gamma=G, **kw)


def uniform(o, q):
    Q = np.empty((5, o.K, o.Np))
    for i in range(5):
        Q[i] = q[i]
    return Q


def jiggle(m, amp, seed):
    """Perturb interior vertices (keeps boundary planes flat) to get general affine tets."""
    rng = np.random.default_rng(seed)
    v = m.vxyz.copy()
    lo, hi = v.min(axis=0), v.max(axis=0)
    interior = np.all((v > lo + 1e-9) & (v < hi - 1e-9), axis=1)
    v[interior] += rng.uniform(-amp, amp, (int(interior.sum()), 3))
    m.vxyz = v
    return m


@pytest.mark.parametrize("N", [1, 2, 3, 4])
def test_free_stream_preservation(N):
    # periodic with a moving uniform state
    m = smesh.kuhn_box((3, 3, 3), (0, 0, 0), (1, 1, 1), periodic=(True, True, True))
    o = om(m, N)
    q = (1.3, 0.2, -0.1, 0.3, 3.0)
    f = rhs(o, uniform(o, q))
    S = np.array([1.4, 1.4, 1.4, 1.4, 2.5])
    hmin = o.geo.h.min()
    assert (np.abs(f).max(axis=(1, 2)) * hmin / S).max() < 1e-12
    # all-wall box at rest, distorted tets
    m = jiggle(smesh.kuhn_box((3, 2, 2), (0, 0, 0), (1, 1, 1), bc_tag=smesh.BC_WALL), 0.05, 1)
    o = om(m, N)
    f = rhs(o, uniform(o, (1.2, 0, 0, 0, 2.7)))
    assert (np.abs(f).max(axis=(1, 2)) * o.geo.h.min() / S).max() < 1e-12
    # pass-through with the ambient ghost state, both lambda modes
    m = jiggle(smesh.kuhn_box((2, 2, 3), (-1, -1, -1), (1, 1, 1)), 0.05, 2)
    for mode in (0, 1):
        o = om(m, N, q_inf=REST, lambda_mode=mode)
        f = rhs(o, uniform(o, REST))
        assert (np.abs(f).max(axis=(1, 2)) * o.geo.h.min() / S).max() < 1e-12
    # inflow faces (Eqs. 5-7) outside the pulse (t >= 2 pi/(alpha tau): p1 = p0) ghost the
    # ambient state: the rest state is preserved; inside the pulse it is not, and only the
    # elements that touch an inflow face feel it at t (one RHS, no propagation yet)
    m = jiggle(smesh.kuhn_box((3, 2, 2), (0, 0, 0), (1, 1, 1), bc_tag=smesh.BC_WALL), 0.05, 3)
    cen = m.vxyz[m.etov[:, smesh.FACES]].mean(axis=2)
    m.bc[(m.bc != 0) & (cen[:, :, 0] < 1e-9)] = smesh.BC_INFLOW
    o = om(m, N, q_inf=REST, inflow_time_scale=1.0)
    f = rhs(o, uniform(o, REST), t=2 * np.pi / 565.0 + 1e-6)
    assert (np.abs(f).max(axis=(1, 2)) * o.geo.h.min() / S).max() < 1e-12
    f = rhs(o, uniform(o, REST), t=np.pi / 565.0)
    touched = (m.bc == smesh.BC_INFLOW).any(axis=1)
    assert np.abs(f[:, touched]).max() > 1e-3 and np.abs(f[:, ~touched]).max() < 1e-12


def _pulse_state(o, seed, vel=0.05, amp=0.05):
    rng = np.random.default_rng(seed)
    x = o.x
    c = rng.uniform(0.3, 0.7, 3)
    bump = amp * np.exp(-((x[0] - c[0]) ** 2 + (x[1] - c[1]) ** 2 + (x[2] - c[2]) ** 2) / 0.1)
    rho = 1.4 * (1 + bump)
    u = vel * np.sin(2 * np.pi * x[1]) + 0.01
    v = vel * np.cos(2 * np.pi * x[2])
    w = vel * np.sin(2 * np.pi * x[0])
    p = 1.0 + bump
    E = p / (G - 1) + 0.5 * rho * (u * u + v * v + w * w)
    return np.stack([rho, rho * u, rho * v, rho * w, E])


def _totals(o, f):
    w = o.ref.M.sum(axis=0)                   # w = M 1
    import math as _m
    tot = [_m.fsum((o.geo.J[:, None] * w[None, :] * f[q]).ravel()) for q in range(5)]
    mag = [_m.fsum((o.geo.J[:, None] * w[None, :] * np.abs(f[q])).ravel()) for q in range(5)]
    return np.array(tot), np.array(mag)


@pytest.mark.parametrize("N", [1, 2, 3])
def test_discrete_conservation(N):
    m = smesh.kuhn_box((3, 3, 3), (0, 0, 0), (1, 1, 1), periodic=(True, True, True))
    o = om(m, N)
    tot, mag = _totals(o, rhs(o, _pulse_state(o, N)))
    assert np.all(np.abs(tot) <= 1e-12 * mag + 1e-300)
    # all-wall box: mass and energy conserved, momentum not (pressure force on the walls)
    m = jiggle(smesh.kuhn_box((3, 3, 2), (0, 0, 0), (1, 1, 1), bc_tag=smesh.BC_WALL), 0.04, 3)
    o = om(m, N)
    tot, mag = _totals(o, rhs(o, _pulse_state(o, N + 10)))
    assert abs(tot[0]) <= 1e-12 * mag[0] and abs(tot[4]) <= 1e-12 * mag[4]
    assert np.abs(tot[1:4]).max() > 1e-6 * mag[1:4].max()


@pytest.mark.parametrize("N", [2, 3])
def test_rotation_covariance(N):
    rng = np.random.default_rng(7)
    Rm, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    if np.linalg.det(Rm) < 0:
        Rm[:, 0] *= -1
    m = smesh.kuhn_box((2, 2, 2), (0, 0, 0), (1, 1, 1), bc_tag=smesh.BC_WALL)
    m.bc[0, :] = np.where(m.bc[0] != 0, smesh.BC_PASSTHROUGH, 0)
    o1 = om(m, N, q_inf=REST)
    Q = _pulse_state(o1, 5, vel=0.1)
    f1 = rhs(o1, Q)
    m2 = smesh.TetMesh(vxyz=m.vxyz @ Rm.T, etov=m.etov, etoe=m.etoe, etof=m.etof, bc=m.bc)
    o2 = om(m2, N, q_inf=REST)
    Q2 = Q.copy()
    Q2[1:4] = np.einsum("ij,jkn->ikn", Rm, Q[1:4])
    f2 = rhs(o2, Q2)
    scale = np.abs(f1).max()
    assert np.abs(f2[0] - f1[0]).max() < 1e-12 * scale
    assert np.abs(f2[4] - f1[4]).max() < 1e-12 * scale
    assert np.abs(f2[1:4] - np.einsum("ij,jkn->ikn", Rm, f1[1:4])).max() < 1e-12 * scale


def _weak_form_rhs(o, Q, nq):
    """Brute force: M_phys dq/dt = int grad(l_i).F_h - sum_f int l_i F*_h  (eq:dgma)."""
    ref, g = o.ref, o.geo
    N, Np, Nfp = o.order, o.Np, o.Nfp
    r, s, t, w = quad.tet_rule(nq)
    L = quad.lagrange_eval(N, ref.r, ref.s, ref.t, r, s, t)
    dL = [quad.lagrange_eval(N, ref.r, ref.s, ref.t, r, s, t, deriv=d) for d in range(3)]
    u2, v2, w2 = quad.tri_rule(nq)
    Mref = L.T @ (w[:, None] * L)
    vM, vP = o.vmaps()
    Qf = Q.reshape(5, -1)
    out = np.zeros_like(Q)
    for k in range(o.K):
        F, Gy, H = euler.euler_fluxes(Q[:, k], G)            # nodal fluxes (5, Np)
        Fh = [L @ F.T, L @ Gy.T, L @ H.T]                    # interpolated flux at quad points
        vol = np.zeros((Np, 5))
        for d in range(3):
            dldx = sum(g.rx[k, a, d] * dL[a] for a in range(3))   # (nq, Np)
            vol += dldx.T @ (w[:, None] * Fh[d])
        vol *= g.J[k]
        sur = np.zeros((Np, 5))
        for f in range(4):
            qm = Qf[:, vM[k, f]]
            qp = Qf[:, vP[k, f]].copy()
            n = g.nx[k, f][:, None]
            if o.bc[k, f] == smesh.BC_WALL:
                qp = euler.ghost_wall(qm, n)
            elif o.bc[k, f] == smesh.BC_PASSTHROUGH:
                qp = euler.ghost_passthrough(qm, o.q_inf)
            lam = euler.llf_lambda(qm, qp, n, G).max()
            fs = euler.llf_flux(qm, qp, n, G, lam)             # (5, Nfp) at face nodes
            fr, fs_, ft = quad.face_points(f, u2, v2)
            Lf = quad.lagrange_eval(N, ref.r, ref.s, ref.t, fr, fs_, ft)      # (nq2, Np)
            Lface = Lf[:, ref.Fmask[f]]
            sur += Lf.T @ (w2[:, None] * (Lface @ fs.T)) * g.sJ[k, f]
        out[:, k] = np.linalg.solve(g.J[k] * Mref, vol - sur).T
    return out


@pytest.mark.parametrize("N", [1, 2, 3])
def test_brute_force_weak_form(N):
    # one distorted element with wall and pass-through faces
    v = np.array([[0.0, 0, 0], [1.1, 0.1, -0.05], [0.2, 0.9, 0.1], [0.05, -0.1, 1.2]])
    one = smesh.TetMesh(vxyz=v, etov=np.array([[0, 1, 2, 3]]), etoe=np.zeros((1, 4), int),
                        etof=np.arange(4)[None, :], bc=np.array([[1, 2, 1, 2]], dtype=np.int8))
    o = om(one, N, q_inf=REST)
    Q = _pulse_state(o, 11, vel=0.2)
    assert np.allclose(rhs(o, Q), _weak_form_rhs(o, Q, N + 4), rtol=0, atol=1e-11 * np.abs(rhs(o, Q)).max())
    # two elements sharing a face
    v = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [0.9, 0.8, 0.7]])
    two = smesh.TetMesh(vxyz=v, etov=np.array([[0, 1, 2, 3], [1, 2, 3, 4]]),
                        etoe=None, etof=None, bc=None)
    from oracle import conn
    e, f = conn.connect_by_hashing(two.etov)
    b = conn.is_boundary(e, f)
    two.etoe, two.etof = e, f
    two.bc = np.where(b, np.array([[1, 2, 2, 1], [2, 1, 1, 2]]), 0).astype(np.int8)
    # element 1 must be positively oriented
    o = om(two, N, q_inf=REST)
    Q = _pulse_state(o, 12, vel=0.2)
    ref = rhs(o, Q)
    assert np.allclose(ref, _weak_form_rhs(o, Q, N + 4), rtol=0, atol=1e-11 * np.abs(ref).max())


def test_element_subset_and_blowup():
    cfg = configs.make("C2", scale=0.25)
    m = cfg.mesh
    o = om(m, cfg.order, q_inf=cfg.q_inf)
    Q = configs.initial_state(cfg, o.x)
    full = rhs(o, Q)
    sub = np.array([0, 5, 17, m.K - 1, 100])
    assert np.array_equal(rhs(o, Q, elems=sub), full[:, sub])
    bad = Q.copy()
    bad[4, 17, 3] = 0.0                                  # p < 0 at one node
    with pytest.raises(BlowUp) as ei:
        rhs(o, bad, t=0.25)
    assert ei.value.element == 17 and ei.value.t == 0.25


def _l2(o, e):
    return math.sqrt(float(np.einsum("k,kn,nm,km->", o.geo.J, e, o.ref.M, e)))


def _run(o, Q, T, cfl=0.5):
    lam = 1.0 + 0.6
    dt0 = cfl * o.geo.h.min() / ((o.order + 1) ** 2 * lam)
    n = int(math.ceil(T / dt0))
    Qn, _, t = timestep.integrate(lambda q, tt: rhs(o, q, tt), Q, 0.0, T / n, n)
    return Qn


@pytest.mark.parametrize("N", [1, 2, 3, 4])
def test_h_convergence_density_wave(N):
    """Exact Euler solution rho = rho0 (1 + eps sin 2pi(x - u t)), velocity and p constant
    (an entropy wave; textbook), on a periodic slab of cubic hexes; L2 rate -> N+1."""
    vel = np.array([0.3, 0.2, 0.1])
    eps, T = 0.1, 0.1
    errs = []
    ns = {1: (4, 8, 16), 2: (8, 16), 3: (6, 12), 4: (4, 8, 12)}[N]
    for n in ns:
        m = smesh.kuhn_box((n, 3, 3), (0, 0, 0), (1, 3.0 / n, 3.0 / n), periodic=(True, True, True))
        o = om(m, N)
        x = o.x

        def state(t):
            rho = 1.4 * (1 + eps * np.sin(2 * np.pi * (x[0] - vel[0] * t)))
            E = 1.0 / (G - 1) + 0.5 * rho * (vel @ vel)
            return np.stack([rho, rho * vel[0], rho * vel[1], rho * vel[2], E])

        QT = _run(o, state(0.0), T)
        errs.append(_l2(o, QT[0] - state(T)[0]) / math.sqrt(9.0 / n ** 2))
    rates = np.log(np.array(errs[:-1]) / np.array(errs[1:])) / np.log(np.array(ns[1:]) / np.array(ns[:-1]))
    # Observed: N=1 -> 2.0, N=2 -> 2.6 (3.36 one level finer), N=3 -> 3.45-3.58.  The
    # sharp a-priori bound for upwind-type DG on general meshes is h^(N+1/2)
    # (Johnson-Pitkaranta / Peterson), optimal h^(N+1) is the usual observation; a
    # dropped term or a wrong sign gives rate <= 1.  Pin: N + 1/2 - 0.1 <= rate <= N + 1.5.
    print(f"N={N} rates {rates}")
    assert N + 0.4 <= rates[-1] <= N + 1.5, (errs, rates)


@pytest.mark.parametrize("N", [1, 2])
def test_acoustic_pulse_vs_linear_acoustics(N):
    """Smooth isentropic acoustic pulse (BASELINE.json north_star; SURVEY P-8 ii, P-10):
    a small planar Gaussian pressure pulse at rest splits into two waves moving at
    c0 = 1 (Eq. 3 scaling): p' = A/2 [g(x - t) + g(x + t)] (linear acoustics;
    nonlinear error O(A^2)).  L2 error must fall at a high-order rate, and the
    numerical pulse must match c = 1 better than c = 1 +- 1 %."""
    A, w, T = 1e-6, 0.1, 0.2

    def g(x, shift):
        out = 0.0
        for m in (-1, 0, 1):
            out = out + np.exp(-((x - 0.5 - shift - m) ** 2) / w ** 2)
        return out

    errs = []
    for n in (8, 16):
        m = smesh.kuhn_box((n, 3, 3), (0, 0, 0), (1, 3.0 / n, 3.0 / n), periodic=(True, True, True))
        o = om(m, N)
        x = o.x[0]
        p = 1.0 + A * g(x, 0.0)
        rho = 1.4 * p ** (1 / G)
        z = np.zeros_like(p)
        QT = _run(o, np.stack([rho, z, z, z, p / (G - 1)]), T)
        pT = euler.pressure(QT, G) - 1.0
        exact = lambda c: 0.5 * A * (g(x, c * T) + g(x, -c * T))
        errs.append(_l2(o, pT - exact(1.0)) / A)
        e_lo, e_hi = _l2(o, pT - exact(0.99)) / A, _l2(o, pT - exact(1.01)) / A
    assert errs[-1] < min(e_lo, e_hi)
    rate = math.log(errs[-2] / errs[-1]) / math.log(2)
    assert rate >= N + 0.4, (errs, rate)       # DG wave errors may superconverge (up to 2N+1)
