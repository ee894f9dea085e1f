"""GPU parity: the sm_100a path (through the C ABI) vs the CPU oracle.

Same seeded inputs on both sides (synth/ recipes at the ORACLE's node
coordinates); tolerances from BASELINE.json (tests/parity.py):
  one RHS <= 1e-11 (scaled), 100 LSERK4 steps <= 1e-9.
Sizes: oracle-sized versions of C1-C5 that span several tiles and a ragged
tail, stepped under several stage-grid caps (parity.GRID_CAPS) so every CTA
walks many tiles (the pipelined steady state the bench times); full-size C2-C5
in the bench launch configuration on sampled elements through all five LSERK4
stages; full-size C2 for 100 steps against a committed oracle run
(tests/golden/make_c2_100.py); edge cases (one element, ragged tails, every
boundary kind, lambda modes, Heun, inflow through the stepper), relabelled and
inverted unstructured-style meshes (all 48 reachable face-orientation codes),
blow-up detection, state round trip, and partition invariance (emulated ranks
on one GPU, exchange by device copies, one-launch and interior/boundary split).
"""
import os
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1710_03887_b200 as dg  # noqa: E402
from oracle import timestep  # noqa: E402
from oracle.rhs import OracleMesh  # noqa: E402
from oracle.rhs import rhs as oracle_rhs  # noqa: E402
from synth import configs  # noqa: E402
from synth import mesh as smesh  # noqa: E402

import meshes  # noqa: E402
import parity  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

SMALL = [("C1", 1.0), ("C2", 0.25), ("C3", 0.15), ("C4", 0.1), ("C5", 0.1)]


def solver(cfg, **kw):
    m = cfg.mesh
    return dg.Solver(cfg.order, m.vxyz, m.etov, m.bc, etoe=m.etoe, etof=m.etof, gamma=cfg.gamma,
                     q_inf=cfg.q_inf, **kw)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


@pytest.mark.parametrize("name,scale", SMALL)
@pytest.mark.parametrize("lambda_mode", [0, 1])
def test_rhs_parity_small(name, scale, lambda_mode):
    cfg = configs.make(name, scale=scale)
    o = parity.oracle_mesh(cfg, lambda_mode)
    Q = configs.initial_state(cfg, o.x)
    s = solver(cfg, lambda_mode=lambda_mode)
    s.set_state(Q)
    g = s.rhs(0.0)
    r = oracle_rhs(o, Q)
    err = parity.e_rhs(g, r, parity.scales(cfg))
    parity.record(f"rhs[{name}@{scale},lambda{lambda_mode}]", e_rhs=err)
    assert err <= parity.RHS_TOL, err
    assert dg.dg_launch_count(s.ctx) >= 2


@pytest.mark.parametrize("name,scale", SMALL)
def test_rk_parity_100_steps(name, scale):
    """100 LSERK4 steps <= 1e-9 (BASELINE.json north_star; eq:ode P:415-419), once per grid cap:
    the default grid (<= 1 tile per CTA on these sizes) and capped grids where every CTA walks
    >= 4 tiles through the cross-tile pipeline, with the residual path (a_s != 0) live."""
    cfg = configs.make(name, scale=scale)
    o = parity.oracle_mesh(cfg)
    Q = configs.initial_state(cfg, o.x)
    dt = parity.oracle_dt(o, Q, cfg.cfl)
    Qo, _, t = timestep.integrate(lambda q, tt: oracle_rhs(o, q, tt), Q, 0.0, dt, 100)
    assert parity.tiles_per_cta(cfg.mesh.K, cfg.order, 2) >= 4
    for cap in parity.GRID_CAPS:
        s = solver(cfg)
        s.set_max_ctas(cap)
        s.set_state(Q)
        s.step(dt, 100)
        G = s.get_state()
        err = parity.e_state(G, Qo, parity.scales(cfg))
        parity.record(f"rk100[{name}@{scale}]", cap=cap, e_state=err, e_pert=parity.e_pert(G, Qo, cfg.q_inf),
                      tiles_per_cta=parity.tiles_per_cta(cfg.mesh.K, cfg.order, cap))
        assert err <= parity.STATE_TOL, (cap, err)
        assert abs(s.time - t) < 1e-12 * max(1.0, t)
        s.close()


@pytest.mark.parametrize("cap", [0, 3])
def test_heun_parity(cap):
    cfg = configs.make("C3", scale=0.15)
    o = parity.oracle_mesh(cfg)
    Q = configs.initial_state(cfg, o.x)
    dt = parity.oracle_dt(o, Q, 0.3)
    s = solver(cfg, rk_scheme=dg.DG_RK_HEUN)
    s.set_max_ctas(cap)
    s.set_state(Q)
    s.step(dt, 20)
    Qo, _, _ = timestep.integrate(lambda q, tt: oracle_rhs(o, q, tt), Q, 0.0, dt, 20, scheme="heun")
    assert parity.e_state(s.get_state(), Qo, parity.scales(cfg)) <= parity.STATE_TOL


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6])
def test_every_order_and_boundary_kind(N):
    """Walls, pass-through and an inflow face (NEXT N1) on one distorted box, every order."""
    m = smesh.kuhn_box((3, 2, 2), (0, 0, 0), (1, 0.7, 0.7), bc_tag=smesh.BC_WALL)
    rng = np.random.default_rng(N)
    lo, hi = m.vxyz.min(0), m.vxyz.max(0)
    inner = np.all((m.vxyz > lo + 1e-9) & (m.vxyz < hi - 1e-9), axis=1)
    m.vxyz[inner] += rng.uniform(-0.03, 0.03, (int(inner.sum()), 3))
    cen = m.vxyz[m.etov].mean(axis=1)
    bnd = m.bc != 0
    m.bc[bnd & (cen[:, 0:1] > 0.6)] = smesh.BC_PASSTHROUGH
    m.bc[bnd & (cen[:, 0:1] < 0.2)] = smesh.BC_INFLOW
    cfg = configs.Config("box", N, m, rho0=1.4, p0=1.0, gamma=1.4,
                         pulses=[(0.05, 0.2, (0.5, 0.35, 0.35))], steps=1)
    o = parity.oracle_mesh(cfg, inflow_time_scale=1.0)
    Q = configs.initial_state(cfg, o.x)
    Q[1] += 0.05 * Q[0] * np.sin(3 * o.x[1])          # some flow so every ghost matters
    Q[4] += 0.5 * (Q[1] ** 2) / Q[0]
    s = solver(cfg, inflow_time_scale=1.0)             # alpha = 565 rad per scaled unit
    s.set_state(Q)
    t = 0.002                                           # inside the inflow pulse
    err = parity.e_rhs(s.rhs(t), oracle_rhs(o, Q, t), parity.scales(cfg))
    assert err <= parity.RHS_TOL, err


@pytest.mark.parametrize("K", [1, 7, 33, 65])
def test_ragged_tails(K):
    cfg = configs.make("C2", scale=0.25)
    m = cfg.mesh
    sub = smesh.TetMesh(vxyz=m.vxyz, etov=m.etov[:K], etoe=None, etof=None, bc=None)
    from oracle.conn import connect_by_hashing
    e, f = connect_by_hashing(sub.etov)
    b = (e == np.arange(K)[:, None]) & (f == np.arange(4)[None, :])
    sub.etoe, sub.etof = e, f
    sub.bc = np.where(b, smesh.BC_WALL, 0).astype(np.int8)
    for N in (3, 4):
        c = configs.Config("sub", N, sub, rho0=1.4, p0=1.0, gamma=1.4, pulses=cfg.pulses, steps=1)
        o = parity.oracle_mesh(c)
        Q = configs.initial_state(c, o.x)
        Q[1] += 0.05 * Q[0] * np.sin(5 * o.x[1] + 1)      # flow, so the rhs is not round-off
        Q[3] += 0.03 * Q[0] * np.cos(4 * o.x[0])
        Q[4] += 0.5 * (Q[1] ** 2 + Q[3] ** 2) / Q[0]
        s = solver(c)
        s.set_state(Q)
        assert parity.e_rhs(s.rhs(0.0), oracle_rhs(o, Q), parity.scales(c)) <= parity.RHS_TOL


def test_free_stream_and_state_roundtrip():
    cfg = configs.make("C5", scale=0.1)
    s = solver(cfg)
    K, Np = s.K, s.Np
    Q = np.empty((5, K, Np))
    for q, v in enumerate((1.3, 0.2, -0.1, 0.3, 3.0)):
        Q[q] = v
    s.set_state(Q)
    assert np.array_equal(s.get_state(), Q)              # bitwise round trip
    f = s.rhs(0.0)
    h = dg.dg_get_geometry(s.ctx)["J"]
    assert np.abs(f).max() < 1e-10 and h.min() > 0


def test_blowup_flag_names_the_element():
    cfg = configs.make("C2", scale=0.25)
    o = parity.oracle_mesh(cfg)
    Q = configs.initial_state(cfg, o.x)
    Q[4, 37, 5] = -1.0
    s = solver(cfg)
    s.set_state(Q)
    s.step(1e-4, 1)
    with pytest.raises(dg.DGError) as e:
        dg.dg_check(s.ctx, s.stream)
    assert e.value.status == dg.DG_EBLOWUP and "element 37" in str(e.value)


@pytest.mark.parametrize("name,order", [("C2", 0), ("C3", 0), ("C4", 0), ("C5", 0), ("C4", 1), ("C4", 2)])
def test_full_size_sampled(name, order):
    """Full BASELINE.json size, bench launch configuration; oracle on sampled elements: one RHS,
    then all five LSERK4 stages through dg_stage_compute.  Each stage's input state is read back
    on the sample and its neighbours, the oracle forms f on the sample from it, carries its own
    residual res_s = a_s res_(s-1) + dt f and predicts Q_(s+1) = Q_s + b_s res_s; stages 1-4 run
    the a_s != 0 residual path in the pipelined steady state (~20-70 tiles per CTA).  order = 1,
    2: the C4 mesh at the paper's orders (`bench.py --order N`; N = 1 is the four-lane kernel of
    csrc/lo.cuh, ~83 tiles of 120 elements per CTA through its three tile buffers)."""
    cfg = configs.make(name)
    if order:
        cfg.order = order
        name = f"{name}-N{order}"
    o = parity.oracle_mesh(cfg)
    Q = configs.initial_state(cfg, o.x)
    s = solver(cfg)
    s.set_state(Q)
    K = cfg.mesh.K
    rng = np.random.default_rng(0)
    wall = np.nonzero((cfg.mesh.bc == smesh.BC_WALL).any(axis=1))[0]
    pt = np.nonzero((cfg.mesh.bc == smesh.BC_PASSTHROUGH).any(axis=1))[0]
    # random elements, the 40 with the largest pulse amplitude (so max|rhs| over the sample is
    # the field's, not round-off), wall and pass-through faces, and the ragged tail
    amp = np.abs(Q[4] - cfg.q_inf[4]).max(axis=1)
    hot = np.argsort(amp)[-40:]
    sample = np.unique(np.concatenate([rng.choice(K, 160, replace=False), hot, wall[:24], pt[:24],
                                       np.arange(K - 9, K), np.arange(0, 5)]))
    patch = np.unique(np.concatenate([sample, cfg.mesh.etoe[sample].ravel()]))
    dsample = torch.as_tensor(sample, device=s.device)
    dpatch = torch.as_tensor(patch, device=s.device)
    g = s.rhs(0.0, device=True)[:, dsample].cpu().numpy()
    r = oracle_rhs(o, Q, 0.0, elems=sample)
    S = parity.scales(cfg)
    e0 = parity.e_rhs(g, r, S)
    parity.record(f"full_rhs[{name}]", e_rhs=e0, sample=len(sample))
    assert e0 <= parity.RHS_TOL
    dt = parity.oracle_dt(o, Q, cfg.cfl)
    Qh = np.zeros_like(Q)
    Qh[:, patch] = Q[:, patch]
    res = np.zeros((5, len(sample), o.Np))
    pos = np.searchsorted(patch, sample)
    for st in range(5):
        f = oracle_rhs(o, Qh, timestep.LSERK4_C[st] * dt, elems=sample)
        res = timestep.LSERK4_A[st] * res + dt * f
        want = Qh[:, sample] + timestep.LSERK4_B[st] * res
        dg.dg_stage_compute(s.ctx, st, dt, 3, s.stream)
        dg.dg_stage_finish(s.ctx, st, dt)
        Qp = s.get_state(device=True)[:, dpatch].cpu().numpy()
        err = parity.e_state(Qp[:, pos], want, S)
        parity.record(f"full_stage[{name}]", stage=st, e_state=err)
        assert err <= 1e-13, (st, err)
        Qh[:, patch] = Qp
    assert abs(s.time - dt) < 1e-15


def test_c2_full_size_100_steps_golden():
    """Full-size C2 (24,576 tets, ~10 tiles per CTA at the default grid) for 100 LSERK4 steps
    through dg_rk_step (CUDA-graph replay), against the committed oracle run
    tests/golden/c2_lserk4_100.npz: the final state of 512 elements (<= 1e-9) and full-field
    properties of the whole GPU state (mass, energy, max deviation from ambient); then again
    with the grid capped at 7 CTAs (~220 tiles per CTA)."""
    gold = np.load(os.path.join(GOLDEN, "c2_lserk4_100.npz"))
    cfg = configs.make("C2")
    o = parity.oracle_mesh(cfg)
    Q = configs.initial_state(cfg, o.x)
    S = parity.scales(cfg)
    wts = o.ref.M.sum(axis=1)
    qinf = np.asarray(cfg.q_inf)[:, None, None]
    for cap in (0, 7):
        s = solver(cfg)
        s.set_max_ctas(cap)
        s.set_state(Q)
        s.step(float(gold["dt"]), int(gold["nsteps"]))
        G = s.get_state()
        assert abs(s.time - float(gold["t_end"])) < 1e-13
        err = parity.e_state(G[:, gold["elems"]], gold["Q_elems"], S)
        parity.record("c2_golden_100", cap=cap, e_state=err,
                      e_pert=parity.e_pert(G[:, gold["elems"]], gold["Q_elems"], cfg.q_inf))
        assert err <= parity.STATE_TOL, (cap, err)
        mass = np.sum(o.geo.J[:, None] * wts[None, :] * G[0])
        energy = np.sum(o.geo.J[:, None] * wts[None, :] * G[4])
        assert abs(mass - float(gold["mass"])) <= 1e-12 * abs(float(gold["mass"]))
        assert abs(energy - float(gold["energy"])) <= 1e-12 * abs(float(gold["energy"]))
        dev = np.abs(G - qinf).reshape(5, -1).max(axis=1)
        assert np.all(np.abs(dev - gold["dev_max"]) <= parity.STATE_TOL * S)
        s.close()


@pytest.mark.parametrize("name,scale", [("C2", 0.25), ("C4", 0.1), ("C5", 0.1)])
def test_relabelled_meshes(name, scale):
    """Unstructured-style local vertex orders (all 48 reachable face-orientation codes,
    tests/meshes.py): one RHS <= 1e-11, 10 LSERK4 steps <= 1e-9 with every CTA walking tiles."""
    cfg = meshes.relabelled(name, scale)
    o = parity.oracle_mesh(cfg)
    Q = configs.initial_state(cfg, o.x)
    Q[1] += 0.02 * Q[0] * np.sin(3 * o.x[2] + 0.5)       # flow, so every trace pairing matters
    Q[4] += 0.5 * Q[1] ** 2 / Q[0]
    S = parity.scales(cfg)
    s = solver(cfg)
    s.set_state(Q)
    assert parity.e_rhs(s.rhs(0.0), oracle_rhs(o, Q), S) <= parity.RHS_TOL
    dt = parity.oracle_dt(o, Q, cfg.cfl)
    Qo, _, _ = timestep.integrate(lambda q, tt: oracle_rhs(o, q, tt), Q, 0.0, dt, 10)
    s.set_max_ctas(3)
    s.step(dt, 10)
    assert parity.e_state(s.get_state(), Qo, S) <= parity.STATE_TOL


@pytest.mark.parametrize("name,scale", [("C2", 0.25), ("C4", 0.1)])
def test_inverted_mesh_repair(name, scale):
    """About half the tets inverted, mixed wall / pass-through tags, connectivity left to the
    library (etoe = NULL): repaired by the S:89 vertex swap with the f1/f3 tags moved along
    (include/dg.h); the oracle runs on its own repair of the same input."""
    from oracle import geom as ogeom
    from oracle.conn import connect_by_hashing
    cfg = meshes.inverted(name, scale)
    m = cfg.mesh
    etov, bc, _ = ogeom.repair_orientation(m.vxyz, m.etov, m.bc)
    etoe, etof = connect_by_hashing(etov)
    o = OracleMesh(order=cfg.order, vxyz=m.vxyz, etov=etov, bc=bc, etoe=etoe, etof=etof,
                   gamma=cfg.gamma, q_inf=cfg.q_inf)
    Q = configs.initial_state(cfg, o.x)
    Q[2] += 0.03 * Q[0] * np.cos(2 * o.x[0] + 0.3)
    Q[4] += 0.5 * Q[2] ** 2 / Q[0]
    s = dg.Solver(cfg.order, m.vxyz, m.etov, m.bc, gamma=cfg.gamma, q_inf=cfg.q_inf)   # etoe = NULL
    assert np.abs(s.nodes() - o.x).max() < 1e-13 * max(1.0, np.abs(o.x).max())
    s.set_state(Q)
    S = parity.scales(cfg)
    assert parity.e_rhs(s.rhs(0.0), oracle_rhs(o, Q), S) <= parity.RHS_TOL
    dt = parity.oracle_dt(o, Q, cfg.cfl)
    Qo, _, _ = timestep.integrate(lambda q, tt: oracle_rhs(o, q, tt), Q, 0.0, dt, 10)
    s.set_max_ctas(2)
    s.step(dt, 10)
    assert parity.e_state(s.get_state(), Qo, S) <= parity.STATE_TOL


def inflow_box(N, seed=1):
    """Distorted box: inflow faces at x = 0 (the paper's mouthpiece), pass-through at
    x = 1, walls elsewhere."""
    m = smesh.kuhn_box((4, 2, 2), (0, 0, 0), (1, 0.5, 0.5), bc_tag=smesh.BC_WALL)
    rng = np.random.default_rng(seed)
    lo, hi = m.vxyz.min(0), m.vxyz.max(0)
    inner = np.all((m.vxyz > lo + 1e-9) & (m.vxyz < hi - 1e-9), axis=1)
    m.vxyz[inner] += rng.uniform(-0.02, 0.02, (int(inner.sum()), 3))
    cen = m.vxyz[m.etov[:, smesh.FACES]].mean(axis=2)
    bnd = m.bc != 0
    m.bc[bnd & (cen[:, :, 0] > 1 - 1e-9)] = smesh.BC_PASSTHROUGH
    m.bc[bnd & (cen[:, :, 0] < 1e-9)] = smesh.BC_INFLOW
    return configs.Config("inflow-box", N, m, rho0=1.4, p0=1.0, gamma=1.4, pulses=[], steps=1)


@pytest.mark.parametrize("rk", ["lserk4", "heun"])
@pytest.mark.parametrize("N", [1, 2, 4])
def test_inflow_through_the_stepper(rk, N):
    """The time-dependent inflow ghost (Eqs. 5-7; reading A24) evaluated at each
    stage time t + c_s dt inside dg_rk_step (reading A20): 40 steps with the pulse duration
    2 pi / (alpha tau) set to 25 dt, so the run covers the rising and falling pulse and the
    switch-off at t = 2 pi / (alpha tau)."""
    cfg = inflow_box(N)
    tau = 1.0
    o0 = parity.oracle_mesh(cfg)
    Q = configs.initial_state(cfg, o0.x)
    dt = parity.oracle_dt(o0, Q, 0.4)
    alpha = 2 * np.pi / (25 * dt * tau)
    kw = dict(inflow_alpha=alpha, inflow_time_scale=tau)
    o = parity.oracle_mesh(cfg, **kw)
    scheme = dg.DG_RK_HEUN if rk == "heun" else dg.DG_RK_LSERK4
    s = solver(cfg, rk_scheme=scheme, **kw)
    s.set_max_ctas(1)
    s.set_state(Q)
    s.step(dt, 40)
    Qo, _, _ = timestep.integrate(lambda q, tt: oracle_rhs(o, q, tt), Q, 0.0, dt, 40, scheme=rk)
    S = parity.scales(cfg)
    assert np.abs(Qo - Q).max() > 1e-3                 # the pulse entered the domain
    assert parity.e_state(s.get_state(), Qo, S) <= parity.STATE_TOL


def ws_view(sv, ptr, nbytes):
    off = ptr - sv.ws.data_ptr()
    assert 0 <= off and off + nbytes <= sv.ws.numel()
    return sv.ws[off:off + nbytes]


@pytest.mark.parametrize("name,scale", [("C4", 0.12), ("C2", 0.5), ("C1", 1.0)])
@pytest.mark.parametrize("nparts,split,cap", [(2, False, 0), (3, False, 0), (2, True, 0), (3, True, 2)])
def test_partition_invariance_emulated(nparts, split, cap, name, scale):
    """P ranks emulated as P contexts on one GPU, halo records exchanged by device copies
    between the stage-level calls: final state bitwise equal to P = 1.  split: the
    production order of dg_rk_step -- pack, interior launch (which = 1) BEFORE the halo
    arrives, then the boundary launch (which = 2, the range starting at K_int) -- and the
    same for dg_rhs_compute; cap: every CTA walks several tiles of each range.  N = 4 (C4),
    N = 3 (C2: dense face segments, level-by-level gathers from the halo records) and N = 2 on
    a periodic mesh (C1: the slabs wrap around)."""
    partition_case(configs.make(name, scale=scale), nparts, split, cap)


def partition_case(cfg, nparts, split, cap):
    o = parity.oracle_mesh(cfg)
    Q = configs.initial_state(cfg, o.x)
    dt = parity.oracle_dt(o, Q, 0.5)
    ref = solver(cfg)
    ref.set_state(Q)
    ref.step(dt, 10)
    want = ref.get_state()
    part = smesh.x_slab_partition(cfg.mesh, nparts)
    ranks = [solver(cfg, part=part, nparts=nparts, rank=r) for r in range(nparts)]
    for r, sv in enumerate(ranks):
        sv.set_max_ctas(cap)
        sv.set_state(Q[:, part == r])
    rec = 5 * ranks[0].Nfp

    def exchange():
        for r, sv in enumerate(ranks):
                npeer, _, _ = dg.dg_halo_info(sv.ctx)
                _, rbuf = dg.dg_halo_buffers(sv.ctx)
                for p in range(npeer):
                    info = dg.dg_halo_peer(sv.ctx, p)
                    other = ranks[info["rank"]]
                    sbuf, _ = dg.dg_halo_buffers(other.ctx)
                    back = [dg.dg_halo_peer(other.ctx, q) for q in range(dg.dg_halo_info(other.ctx)[0])]
                    mine = [b for b in back if b["rank"] == r][0]
                    assert mine["nsend"] == info["nrecv"]
                    n = info["nrecv"] * rec * 8
                    if n:   # device-to-device copy through torch views of the two workspaces
                        dst = ws_view(sv, rbuf + info["recv_off"] * rec * 8, n)
                        src = ws_view(other, sbuf + mine["send_off"] * rec * 8, n)
                        dst.copy_(src)

    # one RHS first (dg_rhs_compute, split or not) against the single-partition RHS
    ref.set_state(Q)
    f_ref = ref.rhs(0.0)
    for sv in ranks:
        dg.dg_stage_pack(sv.ctx, sv.stream)
    outs = [torch.zeros((5, sv.K, sv.Np), dtype=torch.float64, device=sv.device) for sv in ranks]
    if split:
        for sv, o_ in zip(ranks, outs):
            dg.dg_rhs_compute(sv.ctx, 0.0, o_.data_ptr(), 1, sv.stream)
        exchange()
        for sv, o_ in zip(ranks, outs):
            dg.dg_rhs_compute(sv.ctx, 0.0, o_.data_ptr(), 2, sv.stream)
    else:
        exchange()
        for sv, o_ in zip(ranks, outs):
            dg.dg_rhs_compute(sv.ctx, 0.0, o_.data_ptr(), 3, sv.stream)
    f_got = np.empty_like(f_ref)
    for r, o_ in enumerate(outs):
        f_got[:, part == r] = o_.cpu().numpy()
    assert np.array_equal(f_got, f_ref)
    for _ in range(10):
        for st in range(5):
            for sv in ranks:
                dg.dg_stage_pack(sv.ctx, sv.stream)
            if split:
                for sv in ranks:        # interior elements never read the halo
                    dg.dg_stage_compute(sv.ctx, st, dt, 1, sv.stream)
                exchange()
                for sv in ranks:
                    dg.dg_stage_compute(sv.ctx, st, dt, 2, sv.stream)
            else:
                exchange()
                for sv in ranks:
                    dg.dg_stage_compute(sv.ctx, st, dt, 3, sv.stream)
            for sv in ranks:
                dg.dg_stage_finish(sv.ctx, st, dt)
    got = np.empty_like(want)
    for r, sv in enumerate(ranks):
        got[:, part == r] = sv.get_state()
    assert np.array_equal(got, want)


@pytest.mark.parametrize("rk,cap", [(dg.DG_RK_LSERK4, 0), (dg.DG_RK_HEUN, 0), (dg.DG_RK_LSERK4, 3)])
def test_graph_replay_is_bitwise_eager(rk, cap, monkeypatch):
    """dg_rk_step replays captured steps as CUDA graphs on one partition; the result must be
    bit-identical to eager launches, across a dt change (graph re-capture) and both integrators."""
    cfg = configs.make("C2", scale=0.25)
    outs = []
    for eager in (False, True):
        if eager:
            monkeypatch.setenv("DG_NO_GRAPHS", "1")
        else:
            monkeypatch.delenv("DG_NO_GRAPHS", raising=False)
        s = solver(cfg, rk_scheme=rk)
        s.set_max_ctas(cap)
        s.set_state(configs.initial_state(cfg, s.nodes()))
        dt = s.stable_dt(0.4)
        s.step(dt, 7)
        s.step(0.5 * dt, 4)
        outs.append((s.get_state(), s.time))
        s.close()
    assert np.array_equal(outs[0][0], outs[1][0])
    assert outs[0][1] == outs[1][1]
