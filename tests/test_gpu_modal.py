"""GPU parity of the paper's modal-quadrature scheme:
the sm_100a modal stage kernel through the C ABI (scheme = DG_SCHEME_MODAL) vs the oracle's
independent weak-form implementation (oracle/modal.py), on the same seeded nodal inputs.
State and rhs are compared as nodal values (the ABI's representation for both schemes)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1710_03887_b200 as dg  # noqa: E402
from oracle import modal, timestep  # noqa: E402
from synth import configs  # noqa: E402
from synth import mesh as smesh  # noqa: E402

import parity  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def _case(p, seed, periodic=False):
    if periodic:
        m = smesh.kuhn_box((3, 3, 3), (0, 0, 0), (1, 1, 1), periodic=(True, True, True))
    else:
        m = smesh.kuhn_box((3, 2, 2), (0, 0, 0), (1, 0.7, 0.7), bc_tag=smesh.BC_WALL)
        rng = np.random.default_rng(seed)
        lo, hi = m.vxyz.min(0), m.vxyz.max(0)
        inner = np.all((m.vxyz > lo + 1e-9) & (m.vxyz < hi - 1e-9), axis=1)
        m.vxyz[inner] += rng.uniform(-0.03, 0.03, (int(inner.sum()), 3))
        cen = m.vxyz[m.etov].mean(axis=1)
        bnd = m.bc != 0
        m.bc[bnd & (cen[:, 0:1] > 0.6)] = smesh.BC_PASSTHROUGH
        m.bc[bnd & (cen[:, 0:1] < 0.2)] = smesh.BC_INFLOW
    cfg = configs.Config("box", p, m, rho0=1.4, p0=1.0, gamma=1.4,
                         pulses=[(0.05, 0.2, (0.5, 0.35, 0.35))], steps=1)
    return cfg


def _solver(cfg, **kw):
    m = cfg.mesh
    return dg.Solver(cfg.order, m.vxyz, m.etov, m.bc, etoe=m.etoe, etof=m.etof, gamma=cfg.gamma,
                     q_inf=cfg.q_inf, scheme=dg.DG_SCHEME_MODAL, **kw)


def _state(o, cfg):
    Q = configs.initial_state(cfg, o.m.x)
    Q[1] += 0.05 * Q[0] * np.sin(3 * o.m.x[1])
    Q[3] += 0.03 * Q[0] * np.cos(4 * o.m.x[0])
    Q[4] += 0.5 * (Q[1] ** 2 + Q[3] ** 2) / Q[0]
    return Q


@pytest.mark.parametrize("p", [1, 2, 3])
@pytest.mark.parametrize("lambda_mode", [0, 1])
@pytest.mark.parametrize("periodic", [False, True])
def test_modal_rhs_parity(p, lambda_mode, periodic):
    cfg = _case(p, p, periodic)
    o = modal.ModalOracle(parity.oracle_mesh(cfg, lambda_mode, inflow_time_scale=1.0))
    Q = _state(o, cfg)
    s = _solver(cfg, lambda_mode=lambda_mode, inflow_time_scale=1.0)   # alpha per scaled unit
    s.set_state(Q)
    t = 0.002
    want = o.to_nodal(o.rhs(o.to_modal(Q), t))
    err = parity.e_rhs(s.rhs(t), want, parity.scales(cfg))
    assert err <= parity.RHS_TOL, err
    assert np.abs(s.get_state() - Q).max() < 1e-13 * np.abs(Q).max()   # interpolation round trip
    s.close()


@pytest.mark.parametrize("cap", [0, 1])
def test_modal_rk_parity_100_steps(cap):
    cfg = _case(2, 7, periodic=True)
    o = modal.ModalOracle(parity.oracle_mesh(cfg))
    Q = _state(o, cfg)
    dt = 0.5 * parity.oracle_dt(o.m, Q, 0.5)
    s = _solver(cfg)
    s.set_max_ctas(cap)
    s.set_state(Q)
    s.step(dt, 100)
    c, _, _ = timestep.integrate(lambda cc, tt: o.rhs(cc, tt), o.to_modal(Q), 0.0, dt, 100)
    err = parity.e_state(s.get_state(), o.to_nodal(c), parity.scales(cfg))
    assert err <= parity.STATE_TOL, err
    s.close()


def test_modal_sensors_and_dt():
    cfg = _case(2, 3, periodic=True)
    o = modal.ModalOracle(parity.oracle_mesh(cfg))
    Q = _state(o, cfg)
    s = _solver(cfg)
    s.set_state(Q)
    pts = np.array([[0.31, 0.52, 0.47], [0.8, 0.1, 0.9]])
    s.set_sensors(pts)
    got = s.sample_sensors()
    from oracle import sensors
    for i, pt in enumerate(pts):
        k, r, ss, t = sensors.locate(cfg.mesh.vxyz, cfg.mesh.etov, pt)
        want = sensors.sample(2, Q, k, r, ss, t, cfg.gamma)
        assert np.abs(got[i] - want).max() < 1e-12
    assert abs(s.stable_dt(0.5) - parity.oracle_dt(o.m, Q, 0.5)) < 1e-12
    s.close()


@pytest.mark.parametrize("rk", ["lserk4", "heun"])
@pytest.mark.parametrize("p", [1, 2, 3])
def test_modal_inflow_through_the_stepper(rk, p):
    """The inflow ghost at every stage time (reading A20) in the modal scheme: 30 steps with the
    pulse lasting 20 dt (rise, fall and switch-off inside the run)."""
    cfg = _case(p, 5)
    o0 = parity.oracle_mesh(cfg)
    Q = _state(modal.ModalOracle(o0), cfg)
    dt = 0.5 * parity.oracle_dt(o0, Q, 0.4)
    kw = dict(inflow_alpha=2 * np.pi / (20 * dt), inflow_time_scale=1.0)
    o = modal.ModalOracle(parity.oracle_mesh(cfg, **kw))
    s = _solver(cfg, rk_scheme=dg.DG_RK_HEUN if rk == "heun" else dg.DG_RK_LSERK4, **kw)
    s.set_state(Q)
    s.step(dt, 30)
    c, _, _ = timestep.integrate(lambda cc, tt: o.rhs(cc, tt), o.to_modal(Q), 0.0, dt, 30, scheme=rk)
    err = parity.e_state(s.get_state(), o.to_nodal(c), parity.scales(cfg))
    assert err <= parity.STATE_TOL, err
    s.close()


@pytest.mark.parametrize("p", [1, 2, 3])
def test_modal_on_the_horn_mesh_multi_tile(p):
    """The benchmark geometry (C4: carved horn with wall faces, pass-through box) at 0.1 scale,
    the grid capped so every CTA walks many tiles of the modal tile kernel (TMA prefetch of the
    next tile, cp.async neighbour gathers, carried-point face tables on the horn's oblique faces):
    one RHS and 5 LSERK4 steps against the oracle."""
    cfg = configs.make("C4", scale=0.1)
    cfg.order = p
    o = modal.ModalOracle(parity.oracle_mesh(cfg))
    Q = _state(o, cfg)
    s = _solver(cfg)
    s.set_max_ctas(4)
    s.set_state(Q)
    want = o.to_nodal(o.rhs(o.to_modal(Q), 0.0))
    err = parity.e_rhs(s.rhs(0.0), want, parity.scales(cfg))
    assert err <= parity.RHS_TOL, err
    dt = 0.5 * parity.oracle_dt(o.m, Q, 0.5)
    s.step(dt, 5)
    c, _, _ = timestep.integrate(lambda cc, tt: o.rhs(cc, tt), o.to_modal(Q), 0.0, dt, 5)
    err = parity.e_state(s.get_state(), o.to_nodal(c), parity.scales(cfg))
    assert err <= parity.STATE_TOL, err
    s.close()
