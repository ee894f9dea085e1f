"""Face orientations of unstructured meshes (VERDICT r1 "What's missing" 3; SURVEY §7 hard
part 6): host-side trace pairing on relabelled meshes, bit-exact against the
oracle's coordinate-matched vmapP, on one partition and across partitions,
and the orientation-repair path with face tags that must move with their faces."""
import numpy as np
import pytest

import paper_1710_03887_b200 as dg
from oracle import geom as ogeom
from oracle.rhs import OracleMesh
from synth import mesh as smesh

import meshes

REACHABLE = 48    # 4 x 4 face pairs x the 3 vertex permutations of matching parity


def oracle_of(cfg, mesh=None):
    m = mesh or cfg.mesh
    return OracleMesh(order=cfg.order, vxyz=m.vxyz, etov=m.etov, bc=m.bc, etoe=m.etoe, etof=m.etof,
                      gamma=cfg.gamma, q_inf=cfg.q_inf)


def test_kuhn_meshes_use_few_codes_relabelled_reach_all():
    from synth import configs
    base = configs.make("C2", scale=0.25)
    assert len(smesh.face_orientation_codes(base.mesh)) == 6
    for name, scale in (("C2", 0.25), ("C4", 0.1), ("C5", 0.1)):
        codes = smesh.face_orientation_codes(meshes.relabelled(name, scale).mesh)
        assert len(codes) == REACHABLE, (name, len(codes))
        assert len({(f, f2) for f, f2, _ in codes}) == 16


def test_odd_permutations_are_the_other_half():
    """With inverted tets allowed all 96 codes occur; a pair of positively oriented tets never
    shows the other parity: the two face orderings of a shared face, each seen from its own
    tet's outward normal, have opposite handedness."""
    from synth import configs
    m = configs.make("C2", scale=0.25).mesh
    allc = smesh.face_orientation_codes(smesh.relabel_vertices(m, 3, even_only=False))
    even = smesh.face_orientation_codes(smesh.relabel_vertices(m, 3, even_only=True))
    assert len(allc) == 96 and even < allc


@pytest.mark.parametrize("name,scale", [("C2", 0.25), ("C4", 0.1), ("C5", 0.1), ("C3", 0.15)])
def test_relabelled_maps_bit_exact(name, scale):
    cfg = meshes.relabelled(name, scale)
    m = cfg.mesh
    ctx = dg.dg_mesh_create(cfg.order, m.vxyz, m.etov, m.bc, etoe=m.etoe, etof=m.etof, gamma=cfg.gamma,
                            q_inf=cfg.q_inf)
    try:
        o = oracle_of(cfg)
        vM, vP = dg.dg_get_maps(ctx)
        oM, oP = o.vmaps()
        assert np.array_equal(vM, oM)
        assert np.array_equal(vP, oP)
        g = dg.dg_get_geometry(ctx)
        assert np.allclose(g["J"], o.geo.J, rtol=1e-13, atol=0)
        assert np.allclose(g["nx"], o.geo.nx, rtol=0, atol=1e-13)
    finally:
        dg.dg_destroy(ctx)


@pytest.mark.parametrize("nparts", [2, 3])
def test_relabelled_partition_maps_bit_exact(nparts):
    """Every rank's trace map -- local neighbours and halo records (-1 - (g Nfp + j)) -- names
    the oracle's vmapP node; the cut faces carry many orientation codes (halo codes 32 + ...)."""
    cfg = meshes.relabelled("C4", 0.12)
    m = cfg.mesh
    part = smesh.x_slab_partition(m, nparts)
    cut_codes = smesh.face_orientation_codes(m, part)
    assert len(cut_codes) >= 24, len(cut_codes)
    o = oracle_of(cfg)
    oM, oP = o.vmaps()
    Np, Fm = o.Np, o.ref.Fmask
    for r in range(nparts):
        ctx = dg.dg_mesh_create(cfg.order, m.vxyz, m.etov, m.bc, etoe=m.etoe, etof=m.etof, gamma=cfg.gamma,
                                q_inf=cfg.q_inf, part=part, nparts=nparts, rank=r)
        try:
            mine = np.nonzero(part == r)[0]                   # public order = ascending global id
            vM, vP = dg.dg_get_maps(ctx)
            _, _, rg, rf = dg.dg_halo_records(ctx)
            Nfp = o.Nfp
            glob = np.empty_like(vP)
            loc = vP >= 0
            glob[loc] = mine[vP[loc] // Np] * Np + vP[loc] % Np
            gi = -1 - vP[~loc]
            rec, j = gi // Nfp, gi % Nfp
            glob[~loc] = rg[rec] * Np + Fm[rf[rec], j]
            assert np.array_equal(glob, oP[mine])
            assert np.array_equal(mine[vM // Np] * Np + vM % Np, oM[mine])
        finally:
            dg.dg_destroy(ctx)


@pytest.mark.parametrize("name,scale", [("C2", 0.25), ("C4", 0.1)])
def test_orientation_repair_moves_tags_with_faces(name, scale):
    """Inverted tets (etoe = NULL): the library swaps local vertices 2 and 3 (include/dg.h)
    and the f1/f3 tags with them; the oracle repairs the same way and must agree on geometry,
    tags (through the ghost kinds) and maps."""
    cfg = meshes.inverted(name, scale)
    m = cfg.mesh
    etov, bc, flip = ogeom.repair_orientation(m.vxyz, m.etov, m.bc)
    assert 0.3 < flip.mean() < 0.7
    ctx = dg.dg_mesh_create(cfg.order, m.vxyz, m.etov, m.bc, gamma=cfg.gamma, q_inf=cfg.q_inf)
    try:
        from oracle.conn import connect_by_hashing
        etoe, etof = connect_by_hashing(etov)
        fixed = smesh.TetMesh(vxyz=m.vxyz, etov=etov, etoe=etoe, etof=etof, bc=bc)
        o = oracle_of(cfg, fixed)
        g = dg.dg_get_geometry(ctx)
        assert g["J"].min() > 0
        assert np.allclose(g["J"], o.geo.J, rtol=1e-13, atol=0)
        assert np.allclose(g["nx"], o.geo.nx, rtol=0, atol=1e-13)
        vM, vP = dg.dg_get_maps(ctx)
        oM, oP = o.vmaps()
        assert np.array_equal(vM, oM) and np.array_equal(vP, oP)
        # a tag left on the wrong face would pair a boundary face with a paired one
        assert set(np.unique(bc[bc != 0])) == {smesh.BC_WALL, smesh.BC_PASSTHROUGH}
    finally:
        dg.dg_destroy(ctx)
