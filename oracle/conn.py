"""Oracle mesh connectivity: EToE/EToF and the nodal trace maps vmapM/vmapP.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows SURVEY §8(c) O3 and SPEC S:52-60:
* EToE/EToF either come from the caller (then checked for symmetry) or are
  derived by hashing each face's sorted vertex triple; a triple shared by more
  than two tets is a non-manifold mesh error.  A boundary face points at
  itself (EToE[k,f] = k, EToF[k,f] = f).
* vmapM[k,f,i] = k Np + Fmask_f[i].
* vmapP[k,f,i] = the unique node j on the neighbour face (k', f') with
  |(x_i - c_{k,f}) - (x_j - c_{k',f'})| < tol * h, c = face centroid -- this
  pairs ordinary interior faces and periodic faces (a pure translation) alike.
* boundary faces: vmapP = vmapM.
"""
from __future__ import annotations

import numpy as np

from .refelem import FACE_VERTS


def connect_by_hashing(etov: np.ndarray):
    """EToE, EToF (K, 4) from shared sorted vertex triples."""
    etov = np.asarray(etov, dtype=np.int64)
    K = etov.shape[0]
    fv = np.sort(etov[:, np.array(FACE_VERTS)], axis=2).reshape(-1, 3)   # (4K, 3)
    order = np.lexsort((fv[:, 2], fv[:, 1], fv[:, 0]))
    s = fv[order]
    same = np.all(s[1:] == s[:-1], axis=1)
    if np.any(same[1:] & same[:-1]):
        raise ValueError("non-manifold mesh: a face is shared by more than two tetrahedra")
    etoe = np.repeat(np.arange(K, dtype=np.int64)[:, None], 4, axis=1)
    etof = np.repeat(np.arange(4, dtype=np.int64)[None, :], K, axis=0)
    a, b = order[:-1][same], order[1:][same]
    etoe.reshape(-1)[a] = b // 4
    etof.reshape(-1)[a] = b % 4
    etoe.reshape(-1)[b] = a // 4
    etof.reshape(-1)[b] = a % 4
    return etoe, etof


def check_symmetric(etoe: np.ndarray, etof: np.ndarray) -> None:
    K = etoe.shape[0]
    k = np.repeat(np.arange(K)[:, None], 4, axis=1)
    f = np.repeat(np.arange(4)[None, :], K, axis=0)
    if np.any((etoe < 0) | (etoe >= K) | (etof < 0) | (etof > 3)):
        raise ValueError("EToE/EToF out of range")
    back_e = etoe[etoe, etof]
    back_f = etof[etoe, etof]
    if np.any(back_e != k) or np.any(back_f != f):
        raise ValueError("EToE/EToF not symmetric")


def is_boundary(etoe: np.ndarray, etof: np.ndarray) -> np.ndarray:
    K = etoe.shape[0]
    return (etoe == np.arange(K)[:, None]) & (etof == np.arange(4)[None, :])


def build_vmaps(x: np.ndarray, vxyz: np.ndarray, etov: np.ndarray, etoe: np.ndarray,
                etof: np.ndarray, Fmask: np.ndarray, h: np.ndarray, elems=None,
                tol: float = 1e-7, chunk: int = 8192):
    """vmapM, vmapP (E, 4, Nfp) flat indices into K*Np, for elements ``elems``."""
    K, Np = x.shape[1], x.shape[2]
    Nfp = Fmask.shape[1]
    elems = np.arange(K) if elems is None else np.asarray(elems, dtype=np.int64)
    fvi = np.array(FACE_VERTS)
    vmapM = elems[:, None, None] * Np + Fmask[None, :, :]
    vmapP = np.empty_like(vmapM)
    V = np.asarray(vxyz, dtype=np.float64)[np.asarray(etov)]     # (K, 4, 3)
    for c0 in range(0, len(elems), chunk):
        e = elems[c0:c0 + chunk]
        nb, nf = etoe[e], etof[e]                                # (E, 4)
        xm = x[:, e[:, None, None], Fmask[None, :, :]]           # (3, E, 4, Nfp)
        xp = x[:, nb[:, :, None], Fmask[nf]]                     # (3, E, 4, Nfp)
        cm = V[e][:, fvi, :].mean(axis=2)                        # (E, 4, 3)
        cp = V[nb[:, :, None], fvi[nf], :].mean(axis=2)          # (E, 4, 3)
        dm = xm - np.moveaxis(cm, 2, 0)[..., None]
        dp = xp - np.moveaxis(cp, 2, 0)[..., None]
        D = np.sqrt(((dm[..., :, None] - dp[..., None, :]) ** 2).sum(axis=0))   # (E,4,Nfp,Nfp)
        j = np.argmin(D, axis=3)
        dmin = np.take_along_axis(D, j[..., None], axis=3)[..., 0]
        scale = h[e][:, None, None]
        if np.any(dmin > tol * scale):
            raise ValueError("unmatched face nodes (mesh error)")
        Ds = np.sort(D, axis=3)
        if Nfp > 1 and np.any(Ds[..., 1] <= tol * scale):
            raise ValueError("ambiguous face-node match (mesh error)")
        vmapP[c0:c0 + chunk] = nb[:, :, None] * Np + np.take_along_axis(Fmask[nf], j, axis=2)
    bnd = is_boundary(etoe, etof)[elems]
    vmapP[bnd] = vmapM[bnd]
    return vmapM, vmapP
