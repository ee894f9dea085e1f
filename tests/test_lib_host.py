"""Host-side checks of the C-ABI library (no GPU needed).

* the shared library loads and exports every symbol include/dg.h declares;
* dg_mesh_create's host logic (independent fp64 reference element, geometry,
  trace pairing, partition/halo lists) agrees with the oracle: nodes and
  operators to 1e-13 relative, vmapM/vmapP bit-exact (integer work);
* error behaviour of the boundary (include/dg.h).
"""
import re
import os

import numpy as np
import pytest

import paper_1710_03887_b200 as dg
from oracle.rhs import OracleMesh
from synth import configs
from synth import mesh as smesh

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "dg.h")).read()
    declared = set(re.findall(r"\b(dg_[a-z_0-9]+)\s*\(", hdr))
    declared -= {"dg_mesh_desc"}
    assert declared == set(dg.SYMBOLS)
    for name in declared:
        assert hasattr(dg._lib, name)
    # and the binding carries the same names
    for name in declared:
        assert callable(getattr(dg, name))


def _ctx(cfg, **kw):
    m = cfg.mesh
    return dg.dg_mesh_create(cfg.order, m.vxyz, m.etov, m.bc, etoe=m.etoe, etof=m.etof, gamma=cfg.gamma,
                             q_inf=cfg.q_inf, **kw)


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6])
def test_reference_operators_match_oracle(N):
    from oracle.refelem import reference_element
    m = smesh.kuhn_box((2, 2, 2), (0, 0, 0), (1, 1, 1))
    ctx = dg.dg_mesh_create(N, m.vxyz, m.etov, m.bc)
    try:
        ops = dg.dg_get_operators(ctx)
        R = reference_element(N)
        for k in ("r", "s", "t"):
            assert np.abs(ops[k] - getattr(R, k)).max() < 1e-14
        for k in ("Dr", "Ds", "Dt", "LIFT"):
            A, B = ops[k], getattr(R, k)
            assert np.abs(A - B).max() < 1e-13 * max(1.0, np.abs(B).max()), k
        assert np.array_equal(ops["Fmask"], R.Fmask)
    finally:
        dg.dg_destroy(ctx)


@pytest.mark.parametrize("name,scale", [("C1", 1.0), ("C2", 0.25), ("C3", 0.15), ("C4", 0.1), ("C5", 0.1)])
def test_geometry_and_maps_match_oracle(name, scale):
    cfg = configs.make(name, scale=scale)
    m = cfg.mesh
    ctx = _ctx(cfg)
    try:
        o = OracleMesh(order=cfg.order, vxyz=m.vxyz, etov=m.etov, bc=m.bc, etoe=m.etoe, etof=m.etof,
                       gamma=cfg.gamma, q_inf=cfg.q_inf)
        K, Np, Nfp = dg.dg_sizes(ctx)
        assert (K, Np, Nfp) == (o.K, o.Np, o.Nfp)
        x = dg.dg_get_nodes(ctx)
        assert np.abs(x - o.x).max() < 1e-13 * max(1.0, np.abs(o.x).max())
        g = dg.dg_get_geometry(ctx)
        assert np.allclose(g["J"], o.geo.J, rtol=1e-13, atol=0)
        assert np.allclose(g["rx"], o.geo.rx, rtol=1e-12, atol=1e-12 * np.abs(o.geo.rx).max())
        assert np.allclose(g["nx"], o.geo.nx, rtol=0, atol=1e-13)
        assert np.allclose(g["Fscale"], o.geo.Fscale, rtol=1e-13, atol=0)
        vM, vP = dg.dg_get_maps(ctx)
        oM, oP = o.vmaps()
        assert np.array_equal(vM, oM)
        assert np.array_equal(vP, oP)                 # bit-exact index work
    finally:
        dg.dg_destroy(ctx)


def test_face_hashing_path_matches_given_connectivity():
    cfg = configs.make("C3", scale=0.1)
    m = cfg.mesh
    a = _ctx(cfg)
    b = dg.dg_mesh_create(cfg.order, m.vxyz, m.etov, m.bc, gamma=cfg.gamma, q_inf=cfg.q_inf)   # derive EToE
    try:
        assert all(np.array_equal(u, v) for u, v in zip(dg.dg_get_maps(a), dg.dg_get_maps(b)))
    finally:
        dg.dg_destroy(a)
        dg.dg_destroy(b)


def test_orientation_repair_and_errors():
    m = smesh.kuhn_box((2, 1, 1), (0, 0, 0), (1, 1, 1))
    etov = m.etov.copy()
    etov[0, [1, 2]] = etov[0, [2, 1]]           # invert element 0
    # no connectivity given: repaired
    ctx = dg.dg_mesh_create(2, m.vxyz, etov, m.bc)
    assert dg.dg_get_geometry(ctx)["J"].min() > 0
    dg.dg_destroy(ctx)
    # connectivity given: rejected
    with pytest.raises(dg.DGError) as e:
        dg.dg_mesh_create(2, m.vxyz, etov, m.bc, etoe=m.etoe, etof=m.etof)
    assert e.value.status == dg.DG_EMESH
    # boundary face without a tag
    bc = m.bc.copy()
    bc[bc == smesh.BC_PASSTHROUGH] = 0
    with pytest.raises(dg.DGError) as e:
        dg.dg_mesh_create(2, m.vxyz, m.etov, bc)
    assert e.value.status == dg.DG_EMESH
    # non-manifold face
    v = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [0, 0, -1], [1, 1, 1]])
    with pytest.raises(dg.DGError) as e:
        dg.dg_mesh_create(1, v, np.array([[0, 1, 2, 3], [0, 2, 1, 4], [0, 1, 2, 5]]), np.full((3, 4), 2))
    assert e.value.status == dg.DG_EMESH
    # degenerate element
    flat = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0]])
    with pytest.raises(dg.DGError) as e:
        dg.dg_mesh_create(1, flat, np.array([[0, 1, 2, 3]]), np.full((1, 4), 1))
    assert e.value.status == dg.DG_EMESH
    # bad arguments (an empty mesh included)
    with pytest.raises(dg.DGError) as e:
        dg.dg_mesh_create(2, np.zeros((0, 3)), np.zeros((0, 4), dtype=np.int64), np.zeros((0, 4), dtype=np.int32))
    assert e.value.status == dg.DG_EARG
    with pytest.raises(dg.DGError) as e:
        dg.dg_mesh_create(0, m.vxyz, m.etov, m.bc)
    assert e.value.status == dg.DG_EARG
    with pytest.raises(dg.DGError) as e:
        dg.dg_mesh_create(dg.DG_MAX_ORDER + 1, m.vxyz, m.etov, m.bc)
    assert e.value.status == dg.DG_EARG
    with pytest.raises(dg.DGError) as e:
        dg.dg_mesh_create(2, m.vxyz, m.etov, m.bc, gamma=1.0)
    assert e.value.status == dg.DG_EARG
    # device calls before a workspace is bound
    ctx = dg.dg_mesh_create(2, m.vxyz, m.etov, m.bc)
    with pytest.raises(dg.DGError) as e:
        dg.dg_rk_step(ctx, 1e-3, 1, 0)
    assert e.value.status == dg.DG_ESTATE
    dg.dg_destroy(ctx)


def test_memory_report_and_workspace():
    cfg = configs.make("C4", scale=0.1)
    ctx = _ctx(cfg)
    try:
        K, Np, Nfp = dg.dg_sizes(ctx)
        rep = dg.dg_memory_report(ctx)
        assert rep["state"] == 2 * K * 5 * Np * 8 and rep["residual"] == K * 5 * Np * 8
        assert dg.dg_workspace_bytes(ctx) >= sum(rep.values())
    finally:
        dg.dg_destroy(ctx)


@pytest.mark.parametrize("nparts", [2, 3])
def test_partition_halo_lists_pair_up(nparts):
    """Rank p's send list to q and q's receive list from p describe the same faces in
    the same order, and every remote face of every rank is covered."""
    cfg = configs.make("C4", scale=0.1)
    m = cfg.mesh
    part = smesh.x_slab_partition(m, nparts)
    ctxs = [_ctx(cfg, part=part, nparts=nparts, rank=r) for r in range(nparts)]
    try:
        K_tot = sum(dg.dg_sizes(c)[0] for c in ctxs)
        assert K_tot == m.K
        peers = {}
        for r, c in enumerate(ctxs):
            n, ns, nr = dg.dg_halo_info(c)
            peers[r] = {dg.dg_halo_peer(c, p)["rank"]: dg.dg_halo_peer(c, p) for p in range(n)}
            assert sum(p["nsend"] for p in peers[r].values()) == ns
            assert sum(p["nrecv"] for p in peers[r].values()) == nr
        for r in range(nparts):
            for q, info in peers[r].items():
                assert peers[q][r]["nrecv"] == info["nsend"]
        # number of cut faces seen from each side
        etoe = m.etoe
        cut = part[etoe] != part[:, None]
        for r in range(nparts):
            assert sum(p["nrecv"] for p in peers[r].values()) == int(cut[part == r].sum())
    finally:
        for c in ctxs:
            dg.dg_destroy(c)


def test_modal_scheme_limits():
    """DG_SCHEME_MODAL: orders 1-3 on one partition (include/dg.h); others refused."""
    m = smesh.kuhn_box((2, 2, 2), (0, 0, 0), (1, 1, 1))
    for N in (1, 2, 3):
        dg.dg_destroy(dg.dg_mesh_create(N, m.vxyz, m.etov, m.bc, scheme=dg.DG_SCHEME_MODAL))
    with pytest.raises(dg.DGError) as e:
        dg.dg_mesh_create(4, m.vxyz, m.etov, m.bc, scheme=dg.DG_SCHEME_MODAL)
    assert e.value.status == dg.DG_EUNSUPPORTED
    part = (np.arange(m.K) % 2).astype(np.int32)
    with pytest.raises(dg.DGError) as e:
        dg.dg_mesh_create(2, m.vxyz, m.etov, m.bc, part=part, nparts=2, scheme=dg.DG_SCHEME_MODAL)
    assert e.value.status == dg.DG_EUNSUPPORTED
    with pytest.raises(dg.DGError):
        dg.dg_mesh_create(2, m.vxyz, m.etov, m.bc, scheme=7)


def test_nccl_cta_reservation_arguments():
    """dg_set_nccl_ctas (SURVEY §8(e) overlap): [0, 64] accepted before dg_comm_init, else DG_EARG."""
    m = smesh.kuhn_box((3, 3, 3), (0, 0, 0), (1, 1, 1), periodic=(True, True, True))
    ctx = dg.dg_mesh_create(2, m.vxyz, m.etov, m.bc, etoe=m.etoe, etof=m.etof)
    try:
        for n in (0, 2, 64):
            dg.dg_set_nccl_ctas(ctx, n)
        for n in (-1, 65):
            with pytest.raises(dg.DGError) as e:
                dg.dg_set_nccl_ctas(ctx, n)
            assert e.value.status == dg.DG_EARG
    finally:
        dg.dg_destroy(ctx)


def test_spectrum_argument_errors():
    """dg_spectrum validates its arguments on the host (no launch): NULL pointers, n < 2, m < 1."""
    for args in ((0, 16, 1, 8, 8), (8, 1, 1, 8, 8), (8, 16, 0, 8, 8), (8, 16, 1, 0, 8), (8, 16, 70000, 8, 8)):
        with pytest.raises(dg.DGError) as e:
            dg.dg_spectrum(args[0], args[1], args[2], args[3], args[4], 0)
        assert e.value.status == dg.DG_EARG
