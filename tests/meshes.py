"""Test meshes with unstructured-style local vertex orders (the paper's domains
are GMSH tetrahedral meshes, whose local vertex order is arbitrary).

The synthetic Kuhn meshes pair faces in only 6 of the (f, f', sigma) face-orientation codes.
Randomly relabelled copies reach all 48 codes a mesh of positively oriented tets can have
(the other 48 of the 4 x 4 x 6 table need one of the two tets
inverted, which the library either rejects or repairs first)."""
import numpy as np

from synth import configs
from synth import mesh as smesh


def relabelled(name, scale, seed=11):
    """A BASELINE config at `scale` with every tet's local vertex order an even random
    permutation (J > 0 kept, EToE/EToF/bc renumbered consistently)."""
    cfg = configs.make(name, scale=scale)
    cfg.mesh = smesh.relabel_vertices(cfg.mesh, seed, even_only=True)
    cfg.name = f"{name}@{scale}-relabelled"
    return cfg


def mixed_tags(mesh):
    """Distinct boundary tags by side (wall on x-min and y-min sides, pass-through elsewhere),
    so a tag that follows the wrong face is seen."""
    lo = mesh.vxyz.min(axis=0)
    cen = mesh.vxyz[mesh.etov[:, smesh.FACES]].mean(axis=2)          # (K, 4, 3) face centroids
    bnd = mesh.bc != 0
    wall = bnd & ((np.abs(cen[:, :, 0] - lo[0]) < 1e-9) | (np.abs(cen[:, :, 1] - lo[1]) < 1e-9))
    bc = np.where(bnd, smesh.BC_PASSTHROUGH, 0).astype(np.int8)
    bc[wall] = smesh.BC_WALL
    mesh.bc = np.where(mesh.bc == smesh.BC_WALL, smesh.BC_WALL, bc).astype(np.int8)  # keep carved walls
    return mesh


def inverted(name, scale, seed=12):
    """Any random permutation per tet (about half the tets inverted, J < 0), mixed boundary
    tags: the input of the library's orientation repair (etoe = NULL)."""
    cfg = configs.make(name, scale=scale)
    cfg.mesh = smesh.relabel_vertices(mixed_tags(cfg.mesh), seed, even_only=False)
    cfg.name = f"{name}@{scale}-inverted"
    return cfg
