"""Synthetic tetrahedral meshes shaped like the paper's workloads.

Input generation only -- none of the DG method's arithmetic lives here (the
oracle and the CUDA library each derive geometry, maps and operators from
these arrays on their own).  Recipes follow SURVEY §8(c) A11-A13, A17 and
§8(d):

* structured hex grid, each hex split into the 6 Kuhn (path) tetrahedra --
  translation invariant, so opposite periodic faces coincide;
* optional cubed-ball radial map x -> x |x|_inf / |x|_2 (C3; tets stay affine);
* optional horn cavity: tets whose centroid (x_c, rho_c) has x_c in [-0.5, 0.5]
  and rho_c < r(x_c) = 0.02 + 0.15 ((x_c + 0.5)/1.0)^3 are removed and the faces
  they expose are tagged WALL (A12);
* EToE/EToF by hashing sorted vertex triples (periodic directions identify
  vertex indices modulo the grid size first).  Boundary faces point at
  themselves.  Face numbering = the ABI's (f0: v1v2v3, f1: v1v2v4, f2: v2v3v4,
  f3: v1v3v4).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from itertools import permutations

import numpy as np

FACES = np.array([[0, 1, 2], [0, 1, 3], [1, 2, 3], [0, 2, 3]])
BC_INTERIOR, BC_WALL, BC_PASSTHROUGH, BC_INFLOW = 0, 1, 2, 3


@dataclass
class TetMesh:
    vxyz: np.ndarray          # (nv, 3) float64
    etov: np.ndarray          # (K, 4) int64
    etoe: np.ndarray          # (K, 4) int64
    etof: np.ndarray          # (K, 4) int64
    bc: np.ndarray            # (K, 4) int8
    period: tuple | None = None   # box lengths for minimum-image ICs (periodic meshes)
    info: dict = field(default_factory=dict)

    @property
    def K(self) -> int:
        return int(self.etov.shape[0])


def _hash_faces(ids: np.ndarray):
    """EToE/EToF from sorted vertex-id triples; boundary faces point at themselves."""
    K = ids.shape[0]
    fv = np.sort(ids[:, FACES], axis=2).reshape(-1, 3)
    order = np.lexsort((fv[:, 2], fv[:, 1], fv[:, 0]))
    s = fv[order]
    same = np.all(s[1:] == s[:-1], axis=1)
    if np.any(same[1:] & same[:-1]):
        raise ValueError("non-manifold synthetic mesh")
    etoe = np.repeat(np.arange(K, dtype=np.int64)[:, None], 4, axis=1)
    etof = np.repeat(np.arange(4, dtype=np.int64)[None, :], K, axis=0)
    a, b = order[:-1][same], order[1:][same]
    etoe.reshape(-1)[a], etof.reshape(-1)[a] = b // 4, b % 4
    etoe.reshape(-1)[b], etof.reshape(-1)[b] = a // 4, a % 4
    return etoe, etof


def kuhn_box(n, lo, hi, periodic=(False, False, False), bc_tag=BC_PASSTHROUGH, mirror=False) -> TetMesh:
    """n = (nx, ny, nz) hexes on the box [lo, hi], 6 Kuhn tets per hex, hex order x fastest.

    mirror: each hex's Kuhn diagonal is reflected per axis by the sign of its centre coordinate
    (octant symmetry), so every tet contains the hex vertex nearest the origin.  The split stays
    conforming (a shared face's diagonal depends only on the flips of the two axes spanning it,
    which both hexes share).  Used under the cubed-ball map (C3), where the plain split puts
    all four vertices of some corner/edge tets on the sphere (flat slivers)."""
    nx, ny, nz = (int(v) for v in n)
    lo, hi = np.asarray(lo, dtype=np.float64), np.asarray(hi, dtype=np.float64)
    for d, p in enumerate(periodic):
        if p and (nx, ny, nz)[d] < 3:
            raise ValueError("periodic directions need at least 3 hexes")
    gx = np.linspace(lo[0], hi[0], nx + 1)
    gy = np.linspace(lo[1], hi[1], ny + 1)
    gz = np.linspace(lo[2], hi[2], nz + 1)
    Z, Y, X = np.meshgrid(gz, gy, gx, indexing="ij")
    vxyz = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)

    def vid(i, j, k):
        return (k * (ny + 1) + j) * (nx + 1) + i

    k3, j3, i3 = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    i3, j3, k3 = i3.ravel(), j3.ravel(), k3.ravel()
    flips = np.zeros((3, i3.size), dtype=np.int64)
    if mirror:   # reflect the local axis where the hex centre lies on the negative side
        for d, (idx, g) in enumerate(((i3, gx), (j3, gy), (k3, gz))):
            flips[d] = (0.5 * (g[idx] + g[idx + 1]) < -1e-12).astype(np.int64)
    tets = []
    for perm in permutations(range(3)):
        c = [np.zeros(3, dtype=np.int64)]
        for ax in perm:
            nxt = c[-1].copy()
            nxt[ax] += 1
            c.append(nxt)
        verts = [vid(i3 + (o[0] ^ flips[0]), j3 + (o[1] ^ flips[1]), k3 + (o[2] ^ flips[2])) for o in c]
        tets.append(np.stack(verts, axis=1))
    etov = np.stack(tets, axis=1).reshape(-1, 4).astype(np.int64)   # hex-major, 6 per hex
    v = vxyz[etov]                                                   # keep positive orientation
    neg = np.linalg.det(np.stack([v[:, 1] - v[:, 0], v[:, 2] - v[:, 0], v[:, 3] - v[:, 0]], axis=1)) < 0
    etov[neg, 1], etov[neg, 2] = etov[neg, 2].copy(), etov[neg, 1].copy()

    # periodic identification for hashing only (coordinates stay unwrapped)
    iv = np.arange(nx + 1)
    jv = np.arange(ny + 1)
    kv = np.arange(nz + 1)
    if periodic[0]:
        iv = iv % nx
    if periodic[1]:
        jv = jv % ny
    if periodic[2]:
        kv = kv % nz
    KK, JJ, II = np.meshgrid(kv, jv, iv, indexing="ij")
    ident = ((KK * (ny + 1) + JJ) * (nx + 1) + II).ravel()
    etoe, etof = _hash_faces(ident[etov])
    K = etov.shape[0]
    bnd = (etoe == np.arange(K)[:, None]) & (etof == np.arange(4)[None, :])
    bc = np.where(bnd, bc_tag, BC_INTERIOR).astype(np.int8)
    period = tuple(float(hi[d] - lo[d]) if periodic[d] else None for d in range(3))
    return TetMesh(vxyz=vxyz, etov=etov, etoe=etoe, etof=etof, bc=bc,
                   period=period if any(periodic) else None,
                   info={"hexes": (nx, ny, nz), "lo": lo.tolist(), "hi": hi.tolist(), "periodic": list(periodic)})


def cubed_ball(mesh: TetMesh, radius: float = 1.0) -> TetMesh:
    """Map the [-1,1]^3 grid vertices radially onto the ball: x -> x |x|_inf / |x|_2 (A11)."""
    v = mesh.vxyz
    n2 = np.linalg.norm(v, axis=1)
    ninf = np.abs(v).max(axis=1)
    scale = np.where(n2 > 0, ninf / np.where(n2 > 0, n2, 1.0), 0.0)
    mesh.vxyz = v * scale[:, None] * radius
    mesh.info["map"] = "cubed_ball"
    return mesh


def horn_radius(x):
    """r(x) = 0.02 + 0.15 ((x + 0.5)/1.0)^3 on [-0.5, 0.5] (BASELINE.json C3/C4)."""
    return 0.02 + 0.15 * ((np.asarray(x) + 0.5) / 1.0) ** 3


def carve_horn(mesh: TetMesh) -> TetMesh:
    """Remove tets inside the horn and tag the exposed faces WALL (A12)."""
    c = mesh.vxyz[mesh.etov].mean(axis=1)
    rho = np.hypot(c[:, 1], c[:, 2])
    inside = (c[:, 0] >= -0.5) & (c[:, 0] <= 0.5) & (rho < horn_radius(c[:, 0]))
    keep = ~inside
    K = mesh.K
    new_id = -np.ones(K, dtype=np.int64)
    new_id[keep] = np.arange(int(keep.sum()))
    etov = mesh.etov[keep]
    etoe_old, etof_old, bc_old = mesh.etoe[keep], mesh.etof[keep], mesh.bc[keep]
    kk = np.arange(etov.shape[0])
    self_e = np.repeat(kk[:, None], 4, axis=1)
    self_f = np.repeat(np.arange(4)[None, :], etov.shape[0], axis=0)
    nb_new = new_id[etoe_old]
    was_bnd = etoe_old == np.nonzero(keep)[0][:, None]
    was_bnd &= etof_old == self_f
    removed_nb = (~was_bnd) & (nb_new < 0)
    etoe = np.where(was_bnd | removed_nb, self_e, nb_new)
    etof = np.where(was_bnd | removed_nb, self_f, etof_old)
    bc = np.where(removed_nb, BC_WALL, bc_old).astype(np.int8)
    out = TetMesh(vxyz=mesh.vxyz, etov=etov, etoe=etoe, etof=etof, bc=bc, period=mesh.period, info=dict(mesh.info))
    out.info["carved"] = int(inside.sum())
    out.info["wall_faces"] = int((bc == BC_WALL).sum())
    return out


def x_slab_partition(mesh: TetMesh, nparts: int) -> np.ndarray:
    """Equal element-count x-slabs: sort by centroid x, ties by element id."""
    cx = mesh.vxyz[mesh.etov][:, :, 0].mean(axis=1)
    order = np.lexsort((np.arange(mesh.K), cx))
    part = np.empty(mesh.K, dtype=np.int32)
    bounds = np.linspace(0, mesh.K, nparts + 1).round().astype(np.int64)
    for p in range(nparts):
        part[order[bounds[p]:bounds[p + 1]]] = p
    return part


# local vertex opposite each face (FACES[f] = the other three) and the face opposite each vertex
OPPOSITE = np.array([3, 2, 0, 1])
FACE_OF_OPPOSITE = np.argsort(OPPOSITE)            # vertex v -> the face not containing it
_PERMS4 = np.array(list(permutations(range(4))))
_EVEN4 = np.array([p for p in _PERMS4 if round(np.linalg.det(np.eye(4)[list(p)])) > 0])


def relabel_vertices(mesh: TetMesh, seed: int, even_only: bool = True) -> TetMesh:
    """Random local vertex order per tet (an unstructured-mesh input, like GMSH output):
    new etov[k][i] = old etov[k][perm_k[i]].  Faces are renumbered consistently (EToE/EToF/bc
    permuted by the induced face map).  even_only keeps every J > 0 (even permutations preserve
    orientation); odd permutations flip J < 0, which the library repairs only when it derives
    the connectivity itself (etoe = NULL)."""
    rng = np.random.default_rng(seed)
    K = mesh.K
    pool = _EVEN4 if even_only else _PERMS4
    perm = pool[rng.integers(0, len(pool), K)]                    # (K, 4)
    inv = np.argsort(perm, axis=1)
    etov = np.take_along_axis(mesh.etov, perm, axis=1)
    # old face f excludes old vertex OPPOSITE[f], whose new local index is inv[OPPOSITE[f]]
    nf = FACE_OF_OPPOSITE[np.take_along_axis(inv, np.broadcast_to(OPPOSITE, (K, 4)), axis=1)]   # (K, 4)
    etoe = np.empty_like(mesh.etoe)
    etof = np.empty_like(mesh.etof)
    bc = np.empty_like(mesh.bc)
    rows = np.arange(K)[:, None]
    k2 = mesh.etoe
    f2new = nf[k2, mesh.etof]
    etoe[rows, nf] = k2
    etof[rows, nf] = f2new
    bc[rows, nf] = mesh.bc
    out = TetMesh(vxyz=mesh.vxyz, etov=etov, etoe=etoe, etof=etof, bc=bc, period=mesh.period, info=dict(mesh.info))
    out.info["relabelled"] = {"seed": seed, "even_only": even_only}
    return out


def face_orientation_codes(mesh: TetMesh, part=None):
    """Set of (f, f2, sigma) over the paired faces (optionally only the faces whose two elements
    lie on different ranks of `part`), sigma = the tuple m -> m' such that vertex m of face f
    of k coincides with vertex m' of face f2 of its neighbour (positions relative to the face
    centroids, so periodic translations pair too).  For coverage counts in the tests."""
    codes = set()
    v = mesh.vxyz[mesh.etov]                                        # (K, 4, 3)
    for k in range(mesh.K):
        for f in range(4):
            k2, f2 = int(mesh.etoe[k, f]), int(mesh.etof[k, f])
            if k2 == k and f2 == f:
                continue
            if part is not None and part[k] == part[k2]:
                continue
            P = v[k, FACES[f]]
            Qv = v[k2, FACES[f2]]
            P = P - P.mean(axis=0)
            Qv = Qv - Qv.mean(axis=0)
            d = np.linalg.norm(P[:, None, :] - Qv[None, :, :], axis=2)
            sig = tuple(int(j) for j in d.argmin(axis=1))
            codes.add((f, f2, sig))
    return codes


def quality(mesh: TetMesh) -> dict:
    """Mesh-quality statistics for the input recipe (SURVEY §7 hard part 7): J = det of the
    affine map from the reference tet (volume 4/3), h = 3 V / max face area, min and
    median, and the minimum dihedral angle in degrees."""
    v = mesh.vxyz[mesh.etov]                                          # (K, 4, 3)
    e1, e2, e3 = v[:, 1] - v[:, 0], v[:, 2] - v[:, 0], v[:, 3] - v[:, 0]
    J = np.einsum("kd,kd->k", e1, np.cross(e2, e3)) / 8.0
    vol = np.abs(J) * 8.0 / 6.0
    areas = []
    normals = []
    for f in FACES:
        a, b, c = v[:, f[0]], v[:, f[1]], v[:, f[2]]
        nrm = np.cross(b - a, c - a)
        areas.append(0.5 * np.linalg.norm(nrm, axis=1))
        normals.append(nrm / np.linalg.norm(nrm, axis=1)[:, None])
    areas = np.stack(areas, axis=1)
    h = 3.0 * vol / areas.max(axis=1)
    # dihedral angle along the edge shared by faces i and j: pi - angle between outward normals
    opp = OPPOSITE
    cen = v.mean(axis=1)
    out = []
    for f, nrm in enumerate(normals):
        fc = v[:, FACES[f]].mean(axis=1)
        sgn = np.sign(np.einsum("kd,kd->k", nrm, fc - cen))
        out.append(nrm * sgn[:, None])
    dmin = np.full(mesh.K, np.pi)
    for i in range(4):
        for j in range(i + 1, 4):
            cosang = np.clip(np.einsum("kd,kd->k", out[i], out[j]), -1, 1)
            dmin = np.minimum(dmin, np.pi - np.arccos(cosang))
    return {"K": int(mesh.K), "J_min": float(J.min()), "J_median": float(np.median(J)),
            "h_min": float(h.min()), "h_median": float(np.median(h)),
            "h_min_over_median": float(h.min() / np.median(h)),
            "min_dihedral_deg": float(np.degrees(dmin.min())), "median_min_dihedral_deg": float(np.degrees(np.median(dmin)))}
