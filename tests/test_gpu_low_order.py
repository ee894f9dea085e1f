"""GPU parity at the paper's own orders, N = 1 and N = 2 (the paper runs p = 1, PAPER.md P:41,
P:103-120), on the BASELINE meshes with the order overridden.

N = 1 runs the one-thread-per-element kernel (csrc/lo.cuh: TMA-streamed tiles of 192 elements,
operator in the constant bank); these cases span several full tiles and a ragged tail of it,
stepped under grid caps so every CTA walks many tiles and both tile buffers are reused, with
walls, pass-through and inflow ghosts, relabelled (unstructured-style) vertex orders, and
emulated partitions (halo records, interior / boundary split launches).  Tolerances as
tests/parity.py: one RHS <= 1e-11 (scaled), 100 LSERK4 steps <= 1e-9."""
import dataclasses

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1710_03887_b200 as dg  # noqa: E402
from oracle import timestep  # noqa: E402
from oracle.rhs import rhs as oracle_rhs  # noqa: E402
from synth import configs  # noqa: E402

import meshes  # noqa: E402
import parity  # noqa: E402
from test_gpu_parity import partition_case, solver  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def at_order(cfg, N):
    return dataclasses.replace(cfg, order=N, name=f"{cfg.name}-N{N}")


def flow(cfg, o):
    Q = configs.initial_state(cfg, o.x)
    Q[1] += 0.04 * Q[0] * np.sin(3 * o.x[1] + 0.2)       # some flow so every trace and ghost matters
    Q[3] += 0.03 * Q[0] * np.cos(2 * o.x[0])
    Q[4] += 0.5 * (Q[1] ** 2 + Q[3] ** 2) / Q[0]
    return Q


@pytest.mark.parametrize("N", [1, 2])
@pytest.mark.parametrize("name,scale", [("C3", 0.15), ("C4", 0.1), ("C5", 0.1)])
@pytest.mark.parametrize("lambda_mode", [0, 1])
def test_low_order_rhs(N, name, scale, lambda_mode):
    """One RHS: 2,048 / 1,296 / 384 elements (10 / 6 / 2 full tiles of 192 and a ragged tail),
    wall + pass-through (C3, C4) and periodic (C5) meshes, both wave-speed modes."""
    cfg = at_order(configs.make(name, scale=scale), N)
    o = parity.oracle_mesh(cfg, lambda_mode=lambda_mode)
    Q = flow(cfg, o)
    s = solver(cfg, lambda_mode=lambda_mode)
    s.set_state(Q)
    assert parity.e_rhs(s.rhs(0.0), oracle_rhs(o, Q), parity.scales(cfg)) <= parity.RHS_TOL


@pytest.mark.parametrize("N", [1, 2])
@pytest.mark.parametrize("name,scale,cap", [("C4", 0.1, 0), ("C4", 0.1, 2), ("C3", 0.15, 3), ("C5", 0.1, 1)])
def test_low_order_100_steps(N, name, scale, cap):
    """100 LSERK4 steps (all five stages, a_s != 0) with capped grids: a CTA walks up to 6 tiles,
    so both tile buffers are refilled behind bulk stores and the ragged tail follows full tiles."""
    cfg = at_order(configs.make(name, scale=scale), N)
    o = parity.oracle_mesh(cfg)
    Q = configs.initial_state(cfg, o.x)
    dt = parity.oracle_dt(o, Q, 0.5)
    s = solver(cfg)
    s.set_max_ctas(cap)
    s.set_state(Q)
    s.step(dt, 100)
    Qo, _, _ = timestep.integrate(lambda q, tt: oracle_rhs(o, q, tt), Q, 0.0, dt, 100)
    assert parity.e_state(s.get_state(), Qo, parity.scales(cfg)) <= parity.STATE_TOL


@pytest.mark.parametrize("N", [1, 2])
def test_low_order_relabelled(N):
    """Unstructured-style local vertex orders (all 48 reachable face-orientation codes)."""
    cfg = at_order(meshes.relabelled("C4", 0.1), N)
    o = parity.oracle_mesh(cfg)
    Q = flow(cfg, o)
    S = parity.scales(cfg)
    s = solver(cfg)
    s.set_state(Q)
    assert parity.e_rhs(s.rhs(0.0), oracle_rhs(o, Q), S) <= parity.RHS_TOL
    dt = parity.oracle_dt(o, Q, cfg.cfl)
    Qo, _, _ = timestep.integrate(lambda q, tt: oracle_rhs(o, q, tt), Q, 0.0, dt, 10)
    s.set_max_ctas(2)
    s.step(dt, 10)
    assert parity.e_state(s.get_state(), Qo, S) <= parity.STATE_TOL


@pytest.mark.parametrize("N", [1, 2])
@pytest.mark.parametrize("nparts,split,cap", [(2, False, 0), (3, True, 2)])
def test_low_order_partition_invariance(N, nparts, split, cap):
    """Emulated ranks (halo records, interior then boundary launches): bitwise equal to P = 1."""
    partition_case(at_order(configs.make("C4", scale=0.12), N), nparts, split, cap)


def test_low_order_graph_replay_bitwise(monkeypatch):
    cfg = at_order(configs.make("C4", scale=0.1), 1)
    outs = []
    for eager in (False, True):
        if eager:
            monkeypatch.setenv("DG_NO_GRAPHS", "1")
        else:
            monkeypatch.delenv("DG_NO_GRAPHS", raising=False)
        s = solver(cfg)
        s.set_max_ctas(2)
        s.set_state(configs.initial_state(cfg, s.nodes()))
        dt = s.stable_dt(0.4)
        s.step(dt, 7)
        s.step(0.5 * dt, 4)
        outs.append(s.get_state())
        s.close()
    assert np.array_equal(outs[0], outs[1])


# ---- the paper's modal-quadrature scheme at p = 1 (csrc/lo.cuh modal_lo4_kernel)
def _modal_solver(cfg, **kw):
    m = cfg.mesh
    return dg.Solver(cfg.order, m.vxyz, m.etov, m.bc, etoe=m.etoe, etof=m.etof, gamma=cfg.gamma,
                     q_inf=cfg.q_inf, scheme=dg.DG_SCHEME_MODAL, **kw)


@pytest.mark.parametrize("name,scale,cap,relabel", [("C4", 0.1, 1, False), ("C4", 0.1, 2, True), ("C3", 0.15, 3, False),
                                                     ("C5", 0.1, 1, False)])
def test_modal_p1_many_tiles(name, scale, cap, relabel):
    """p = 1 modal scheme with every CTA walking 4-11 tiles of 120 elements (all three tile
    buffers refilled behind bulk stores, ragged tail last): one RHS in both wave-speed modes and
    40 LSERK4 steps against the modal oracle; horn meshes with walls and pass-through faces, a
    periodic mesh, and unstructured-style vertex orders (carried-point face tables of every
    reachable orientation code)."""
    from oracle import modal
    cfg = at_order(meshes.relabelled(name, scale) if relabel else configs.make(name, scale=scale), 1)
    S = parity.scales(cfg)
    for lambda_mode in (1, 0):
        o = modal.ModalOracle(parity.oracle_mesh(cfg, lambda_mode))
        Q = flow(cfg, o.m)
        s = _modal_solver(cfg, lambda_mode=lambda_mode)
        s.set_max_ctas(cap)
        s.set_state(Q)
        want = o.to_nodal(o.rhs(o.to_modal(Q), 0.0))
        assert parity.e_rhs(s.rhs(0.0), want, S) <= parity.RHS_TOL
    dt = 0.5 * parity.oracle_dt(o.m, Q, 0.5)
    s.step(dt, 40)
    c, _, _ = timestep.integrate(lambda cc, tt: o.rhs(cc, tt), o.to_modal(Q), 0.0, dt, 40)
    assert parity.e_state(s.get_state(), o.to_nodal(c), S) <= parity.STATE_TOL
    s.close()


@pytest.mark.parametrize("scheme", ["nodal", "modal"])
def test_paper_order_full_size_properties(scheme):
    """Properties that hold at any size, on the full-size meshes in the bench launch configuration
    (one CTA per SM, ~83 / ~22 tiles per CTA), for both p = 1 kernels of csrc/lo.cuh:
    (1) C4 (walls + pass-through): the ambient state is steady -- rhs = 0 up to round-off (the
        ghosts equal the interior state, the wall mirror of zero momentum is itself);
    (2) C5 (periodic): discrete conservation -- sum_k J_k * (element mean of rhs) = 0 for all five
        fields (the mean of a linear polynomial over a tet is the mean of its vertex values; the
        face fluxes cancel pairwise, S:342 / `eq:dgma`), relative to sum_k J_k * mean |rhs|."""
    mk = _modal_solver if scheme == "modal" else solver
    cfg = at_order(configs.make("C4"), 1)
    s = mk(cfg)
    K, Np = s.K, s.Np
    Q = np.empty((5, K, Np))
    for c in range(5):
        Q[c] = cfg.q_inf[c]
    s.set_state(Q)
    f = s.rhs(0.0)
    S = parity.scales(cfg)
    assert (np.abs(f).reshape(5, -1).max(axis=1) / S).max() <= 1e-12
    s.close()
    cfg = at_order(configs.make("C5"), 1)
    o = parity.oracle_mesh(cfg)
    s = mk(cfg)
    Q = configs.initial_state(cfg, s.nodes())
    Q[1] += 0.05 * Q[0] * np.sin(2 * np.pi * s.nodes()[1])     # periodic flow
    Q[4] += 0.5 * Q[1] ** 2 / Q[0]
    s.set_state(Q)
    f = s.rhs(0.0)
    J = o.geo.J
    tot = (J[None, :] * f.mean(axis=2)).sum(axis=1)
    ref = (J[None, :] * np.abs(f).mean(axis=2)).sum(axis=1)
    assert np.all(np.abs(tot) <= 1e-11 * ref.max()), (tot, ref)
    s.close()
