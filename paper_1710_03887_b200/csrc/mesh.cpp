// Host-side mesh processing of dg_mesh_create (library side; no device work).
//
// SPEC S:18-102 (mesh module contract, restated for the ABI) and SURVEY §8(c)
// O2/O3: orientation fix-up, EToE/EToF derivation by face hashing or symmetry
// check, boundary-tag validation, affine geometric factors, trace pairing of
// every interior face (vertex permutation found on coordinates relative to the
// face centroids, so periodic translations pair too, then verified node by
// node), the rank's element set for an element partition and its halo lists.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <tuple>

#include "ctx.h"
#include "refelem.h"

namespace dgb {

namespace {

dg_status fail(dg_ctx* c, dg_status st, const std::string& m) {
  c->err = m;
  return st;
}

struct V3 {
  double x, y, z;
};
inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline double norm(V3 a) { return std::sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }

double det3(const double A[9]) {
  return A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) + A[2] * (A[3] * A[7] - A[4] * A[6]);
}

}  // namespace

dg_status build_ctx(const dg_mesh_desc* d, int rank, dg_ctx* c) {
  if (!d) return fail(c, DG_EARG, "desc is NULL");
  if (d->order < 1 || d->order > DG_MAX_ORDER) return fail(c, DG_EARG, "order must be in [1, DG_MAX_ORDER]");
  if (d->nv <= 0 || d->k <= 0 || !d->vxyz || !d->etov || !d->bc) return fail(c, DG_EARG, "empty mesh or NULL array");
  if ((d->etoe == nullptr) != (d->etof == nullptr)) return fail(c, DG_EARG, "etoe and etof must both be given or both be NULL");
  if (!(d->gamma > 1.0)) return fail(c, DG_EARG, "gamma must be > 1");
  const int nparts = d->part ? d->nparts : 1;
  if (nparts < 1 || rank < 0 || rank >= nparts) return fail(c, DG_EARG, "rank/nparts out of range");
  if (d->k > (int64_t(1) << 31) / 8) return fail(c, DG_EARG, "too many elements for int32 indexing");
  if (d->lambda_mode != 0 && d->lambda_mode != 1) return fail(c, DG_EARG, "lambda_mode must be 0 or 1");
  if (d->rk_scheme != DG_RK_LSERK4 && d->rk_scheme != DG_RK_HEUN) return fail(c, DG_EARG, "unknown rk_scheme");

  c->N = d->order;
  c->rank = rank;
  c->nparts = nparts;
  c->gamma = d->gamma;
  for (int i = 0; i < 5; ++i) c->q_inf[i] = d->q_inf[i];
  c->lambda_mode = d->lambda_mode;
  c->check_every = d->check_every;
  c->rk_scheme = d->rk_scheme;
  c->inflow_alpha = d->inflow_alpha > 0 ? d->inflow_alpha : 565.0;
  c->inflow_time_scale = d->inflow_time_scale > 0 ? d->inflow_time_scale : 2.915e-5;
  c->inflow_half_amplitude = d->inflow_half_amplitude > 0 ? d->inflow_half_amplitude : 0.05;
  if (!std::isfinite(c->inflow_alpha) || !std::isfinite(c->inflow_time_scale) || !std::isfinite(c->inflow_half_amplitude))
    return fail(c, DG_EARG, "inflow parameters must be finite");
  {
    // q_inf: the pass-through ghost (Eq. 3) and the inflow ambient state; its pressure is the
    // background subtracted from the fluxes (A14).  Decided over the whole mesh, so every rank
    // of a partition uses the same pref (bitwise partition invariance).
    const double* q = d->q_inf;
    bool fin = true;
    for (int i = 0; i < 5; ++i) fin &= std::isfinite(q[i]);
    const double p = fin && q[0] > 0 ? (d->gamma - 1.0) * (q[4] - 0.5 * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3]) / q[0]) : 0.0;
    c->qinf_valid = fin && q[0] > 0 && p > 0 && std::isfinite(p);
    c->pref = c->qinf_valid ? p : 0.0;
    bool used = false;
    for (int64_t i = 0; i < 4 * d->k && !used; ++i) used = d->bc[i] == DG_BC_PASSTHROUGH || d->bc[i] == DG_BC_INFLOW;
    if (used && !c->qinf_valid)
      return fail(c, DG_EARG, "q_inf must be a valid state (finite, rho > 0, p > 0): the mesh has pass-through or inflow faces");
  }
  std::string msg;
  if (!build_reference(c->N, c->ref, &msg)) return fail(c, DG_EARG, "reference element: " + msg);
  if (d->scheme != DG_SCHEME_NODAL && d->scheme != DG_SCHEME_MODAL) return fail(c, DG_EARG, "unknown scheme");
  c->scheme = d->scheme;
  if (c->scheme == DG_SCHEME_MODAL) {
    if (c->N > 3) return fail(c, DG_EUNSUPPORTED, "the modal scheme is built for orders 1-3");
    if (nparts > 1) return fail(c, DG_EUNSUPPORTED, "the modal scheme runs on one partition");
    if (!build_modal(c->ref, c->modal, &msg)) return fail(c, DG_EARG, "modal tables: " + msg);
    const ModalTables& T = c->modal;
    for (const std::vector<double>* v : {&T.wq, &T.Vq, &T.Dq, &T.wf, &T.Pstd, &T.Pmap, &T.V, &T.Vinv})
      c->modal_cat.insert(c->modal_cat.end(), v->begin(), v->end());
  }
  const int N = c->N, Np = c->ref.Np, Nfp = c->ref.Nfp;
  c->Np = Np;
  c->Nfp = Nfp;
  const int64_t K = d->k, nv = d->nv;

  // ---- vertices per element, orientation
  std::vector<int64_t> etov(d->etov, d->etov + 4 * K);
  std::vector<int8_t> bcv(d->bc, d->bc + 4 * K);   // tags in the (repaired) face numbering
  for (int64_t i = 0; i < 4 * K; ++i)
    if (etov[i] < 0 || etov[i] >= nv) return fail(c, DG_EMESH, "EToV references an unknown vertex (element " + std::to_string(i / 4) + ")");
  auto vert = [&](int64_t v) { return V3{d->vxyz[3 * v], d->vxyz[3 * v + 1], d->vxyz[3 * v + 2]}; };
  auto jac = [&](int64_t k, double A[9]) {
    V3 v0 = vert(etov[4 * k]), v1 = vert(etov[4 * k + 1]), v2 = vert(etov[4 * k + 2]), v3 = vert(etov[4 * k + 3]);
    V3 a = sub(v1, v0), b = sub(v2, v0), e = sub(v3, v0);
    // columns dx/dr, dx/ds, dx/dt
    A[0] = a.x / 2; A[1] = b.x / 2; A[2] = e.x / 2;
    A[3] = a.y / 2; A[4] = b.y / 2; A[5] = e.y / 2;
    A[6] = a.z / 2; A[7] = b.z / 2; A[8] = e.z / 2;
    return det3(A);
  };
  for (int64_t k = 0; k < K; ++k) {
    double A[9];
    double J = jac(k, A);
    if (!(J > 0)) {
      if (J == 0.0 || !std::isfinite(J)) return fail(c, DG_EMESH, "degenerate element " + std::to_string(k) + " (J = 0)");
      if (d->etoe) return fail(c, DG_EMESH, "element " + std::to_string(k) + " has J <= 0 and connectivity was given");
      std::swap(etov[4 * k + 1], etov[4 * k + 2]);   // S:89 repair
      // the swap exchanges the vertex sets of faces f1 (v1 v2 v4) and f3 (v1 v3 v4): their
      // tags, given in the caller's face numbering, move with them
      std::swap(bcv[4 * k + 1], bcv[4 * k + 3]);
    }
  }

  // ---- connectivity
  std::vector<int64_t> etoe(4 * K);
  std::vector<int8_t> etof(4 * K);
  if (d->etoe) {
    for (int64_t i = 0; i < 4 * K; ++i) {
      etoe[i] = d->etoe[i];
      etof[i] = d->etof[i];
      if (etoe[i] < 0 || etoe[i] >= K || etof[i] < 0 || etof[i] > 3) return fail(c, DG_EMESH, "EToE/EToF out of range");
    }
    for (int64_t k = 0; k < K; ++k)
      for (int f = 0; f < 4; ++f) {
        int64_t k2 = etoe[4 * k + f];
        int f2 = etof[4 * k + f];
        if (etoe[4 * k2 + f2] != k || etof[4 * k2 + f2] != f)
          return fail(c, DG_EMESH, "EToE/EToF not symmetric at element " + std::to_string(k));
      }
  } else {
    std::vector<std::tuple<int64_t, int64_t, int64_t, int64_t>> rec(4 * K);
    for (int64_t k = 0; k < K; ++k)
      for (int f = 0; f < 4; ++f) {
        std::array<int64_t, 3> v = {etov[4 * k + FACE_VERTS[f][0]], etov[4 * k + FACE_VERTS[f][1]], etov[4 * k + FACE_VERTS[f][2]]};
        std::sort(v.begin(), v.end());
        rec[4 * k + f] = {v[0], v[1], v[2], 4 * k + f};
      }
    std::sort(rec.begin(), rec.end());
    for (int64_t i = 0; i < 4 * K; ++i) {
      int64_t id = std::get<3>(rec[i]);
      etoe[id] = id / 4;
      etof[id] = int8_t(id % 4);
    }
    for (int64_t i = 0; i + 1 < 4 * K; ++i) {
      auto same = [&](int64_t a, int64_t b) {
        return std::get<0>(rec[a]) == std::get<0>(rec[b]) && std::get<1>(rec[a]) == std::get<1>(rec[b]) &&
               std::get<2>(rec[a]) == std::get<2>(rec[b]);
      };
      if (same(i, i + 1)) {
        if (i + 2 < 4 * K && same(i, i + 2)) return fail(c, DG_EMESH, "non-manifold face (shared by more than two tetrahedra)");
        int64_t a = std::get<3>(rec[i]), b = std::get<3>(rec[i + 1]);
        etoe[a] = b / 4; etof[a] = int8_t(b % 4);
        etoe[b] = a / 4; etof[b] = int8_t(a % 4);
        ++i;
      }
    }
  }
  for (int64_t k = 0; k < K; ++k)
    for (int f = 0; f < 4; ++f) {
      bool bnd = etoe[4 * k + f] == k && etof[4 * k + f] == f;
      int tag = bcv[4 * k + f];
      if (bnd && (tag < DG_BC_WALL || tag > DG_BC_INFLOW))
        return fail(c, DG_EMESH, "boundary face without a valid tag (element " + std::to_string(k) + ", face " + std::to_string(f) + ")");
      if (!bnd && tag != DG_BC_INTERIOR)
        return fail(c, DG_EMESH, "paired face carries a boundary tag (element " + std::to_string(k) + ")");
    }

  // ---- partition
  std::vector<int32_t> part(K, 0);
  if (d->part)
    for (int64_t k = 0; k < K; ++k) {
      part[k] = d->part[k];
      if (part[k] < 0 || part[k] >= nparts) return fail(c, DG_EARG, "part[] out of range");
    }
  std::vector<int64_t> mine, inter, bound;
  for (int64_t k = 0; k < K; ++k)
    if (part[k] == rank) {
      mine.push_back(k);
      bool b = false;
      for (int f = 0; f < 4; ++f) b |= part[etoe[4 * k + f]] != rank;
      (b ? bound : inter).push_back(k);
    }
  if (mine.empty()) return fail(c, DG_EARG, "rank owns no elements");
  c->K = int64_t(mine.size());
  // the interior range ends on a 32-element boundary so that every stage-kernel tile of the
  // boundary range starts 16-byte aligned for its TMA bulk copies (Q/res: K*5*Np doubles,
  // geo: 25 doubles, code: 4 bytes per element); the few interior elements moved into the
  // boundary range merely wait for the halo
  c->K_int = int64_t(inter.size()) / 32 * 32;
  for (int64_t k : mine)
    for (int f = 0; f < 4; ++f) c->has_inflow |= bcv[4 * k + f] == DG_BC_INFLOW;
  c->gid = inter;
  c->gid.insert(c->gid.end(), bound.begin(), bound.end());
  std::vector<int64_t> g2l(K, -1), g2pub(K, -1);
  for (int64_t i = 0; i < c->K; ++i) g2l[c->gid[i]] = i;
  for (int64_t i = 0; i < c->K; ++i) g2pub[mine[i]] = i;
  c->pub.resize(c->K);
  for (int64_t i = 0; i < c->K; ++i) c->pub[i] = int32_t(g2pub[c->gid[i]]);

  // ---- geometric factors
  const int64_t KL = c->K;
  c->geo.assign(KL * 25, 0.0);
  c->J.resize(KL);
  c->h.resize(KL);
  std::vector<double> nrm(KL * 12);
  for (int64_t l = 0; l < KL; ++l) {
    const int64_t k = c->gid[l];
    double A[9];
    const double J = jac(k, A);
    // inverse Jacobian: rows grad r, grad s, grad t
    double I[9];
    I[0] = (A[4] * A[8] - A[5] * A[7]) / J; I[1] = (A[2] * A[7] - A[1] * A[8]) / J; I[2] = (A[1] * A[5] - A[2] * A[4]) / J;
    I[3] = (A[5] * A[6] - A[3] * A[8]) / J; I[4] = (A[0] * A[8] - A[2] * A[6]) / J; I[5] = (A[2] * A[3] - A[0] * A[5]) / J;
    I[6] = (A[3] * A[7] - A[4] * A[6]) / J; I[7] = (A[1] * A[6] - A[0] * A[7]) / J; I[8] = (A[0] * A[4] - A[1] * A[3]) / J;
    double* G = &c->geo[l * 25];
    for (int i = 0; i < 9; ++i) G[i] = I[i];
    double gr[3] = {I[0], I[1], I[2]}, gs[3] = {I[3], I[4], I[5]}, gt[3] = {I[6], I[7], I[8]};
    double gf[4][3];
    for (int q = 0; q < 3; ++q) {
      gf[0][q] = -gt[q];
      gf[1][q] = -gs[q];
      gf[2][q] = gr[q] + gs[q] + gt[q];
      gf[3][q] = -gr[q];
    }
    double amax = 0;
    for (int f = 0; f < 4; ++f) {
      double gn = std::sqrt(gf[f][0] * gf[f][0] + gf[f][1] * gf[f][1] + gf[f][2] * gf[f][2]);
      for (int q = 0; q < 3; ++q) {
        G[9 + 4 * f + q] = gf[f][q] / gn;
        nrm[l * 12 + 3 * f + q] = gf[f][q] / gn;
      }
      G[9 + 4 * f + 3] = gn;          // Fscale = sJ / J
      amax = std::max(amax, 2.0 * gn * J);
    }
    c->J[l] = J;
    c->h[l] = 3.0 * (4.0 * J / 3.0) / amax;
  }

  // ---- node coordinates
  auto node_xyz = [&](int64_t k, int n) {
    V3 v0 = vert(etov[4 * k]), v1 = vert(etov[4 * k + 1]), v2 = vert(etov[4 * k + 2]), v3 = vert(etov[4 * k + 3]);
    double r = c->ref.r[n], s = c->ref.s[n], t = c->ref.t[n];
    double w0 = -(1 + r + s + t) / 2, w1 = (1 + r) / 2, w2 = (1 + s) / 2, w3 = (1 + t) / 2;
    return V3{w0 * v0.x + w1 * v1.x + w2 * v2.x + w3 * v3.x, w0 * v0.y + w1 * v1.y + w2 * v2.y + w3 * v3.y,
              w0 * v0.z + w1 * v1.z + w2 * v2.z + w3 * v3.z};
  };
  c->xyz.assign(3 * KL * Np, 0.0);
  for (int64_t l = 0; l < KL; ++l) {
    int64_t p = c->pub[l];
    for (int n = 0; n < Np; ++n) {
      V3 x = node_xyz(c->gid[l], n);
      c->xyz[(0 * KL + p) * Np + n] = x.x;
      c->xyz[(1 * KL + p) * Np + n] = x.y;
      c->xyz[(2 * KL + p) * Np + n] = x.z;
    }
  }

  // ---- face pairing: vertex permutation from centroid-relative coordinates
  c->nbr.assign(KL * 4, -1);
  c->code.assign(KL * 4, 0);
  struct Ghost { int peer; int64_t sgid; int sface; int64_t l; int f; int sigma; };
  std::vector<Ghost> ghosts;
  std::map<int, std::vector<std::pair<int64_t, int>>> sends;   // peer -> (my gid, my face)
  auto face_v = [&](int64_t k, int f, V3 (&P)[3], V3& cen) {
    cen = {0, 0, 0};
    for (int m = 0; m < 3; ++m) {
      P[m] = vert(etov[4 * k + FACE_VERTS[f][m]]);
      cen.x += P[m].x / 3; cen.y += P[m].y / 3; cen.z += P[m].z / 3;
    }
  };
  for (int64_t l = 0; l < KL; ++l) {
    const int64_t k = c->gid[l];
    for (int f = 0; f < 4; ++f) {
      const int64_t k2 = etoe[4 * k + f];
      const int f2 = etof[4 * k + f];
      if (k2 == k && f2 == f) {
        c->code[l * 4 + f] = uint8_t(64 + bcv[4 * k + f]);
        continue;
      }
      V3 P[3], Q[3], cP, cQ;
      face_v(k, f, P, cP);
      face_v(k2, f2, Q, cQ);
      double scale = 0;
      for (int m = 0; m < 3; ++m) scale = std::max(scale, norm(sub(P[m], cP)));
      const double tol = 1e-8 * scale;
      int sigma = -1;
      for (int sg = 0; sg < 6; ++sg) {
        double err = 0;
        for (int m = 0; m < 3; ++m) err = std::max(err, norm(sub(sub(P[m], cP), sub(Q[PERM6[sg][m]], cQ))));
        if (err < tol) {
          if (sigma >= 0) return fail(c, DG_EMESH, "ambiguous face pairing (element " + std::to_string(k) + ")");
          sigma = sg;
        }
      }
      if (sigma < 0) return fail(c, DG_EMESH, "unmatched face nodes: element " + std::to_string(k) + " face " + std::to_string(f));
      // node-by-node verification of the pairing
      for (int i = 0; i < Nfp; ++i) {
        int j = c->ref.nbr_local[((f * 4 + f2) * 6 + sigma) * Nfp + i];
        V3 xa = sub(node_xyz(k, c->ref.Fmask[f * Nfp + i]), cP);
        V3 xb = sub(node_xyz(k2, c->ref.Fmask[f2 * Nfp + j]), cQ);
        if (norm(sub(xa, xb)) > 1e-7 * scale) return fail(c, DG_EMESH, "unmatched face nodes: element " + std::to_string(k));
      }
      if (part[k2] == rank) {
        c->nbr[l * 4 + f] = int32_t(g2l[k2]);
        c->code[l * 4 + f] = uint8_t(f2 * 6 + sigma);
      } else {
        ghosts.push_back({part[k2], k2, f2, l, f, sigma});
        sends[part[k2]].push_back({k, f});
      }
    }
  }

  // ---- halo lists: both sides order a peer's records by (sender gid, sender face)
  std::map<int, std::vector<Ghost>> recv_by;
  for (auto& g : ghosts) recv_by[g.peer].push_back(g);
  std::vector<int> peer_ranks;
  for (auto& kv : recv_by) peer_ranks.push_back(kv.first);
  for (auto& kv : sends)
    if (!recv_by.count(kv.first)) peer_ranks.push_back(kv.first);
  std::sort(peer_ranks.begin(), peer_ranks.end());
  int64_t roff = 0, soff = 0;
  for (int q : peer_ranks) {
    dg_peer P{q, soff, 0, roff, 0};
    auto& rv = recv_by[q];
    std::sort(rv.begin(), rv.end(), [](const Ghost& a, const Ghost& b) {
      return a.sgid != b.sgid ? a.sgid < b.sgid : a.sface < b.sface;
    });
    for (size_t i = 0; i < rv.size(); ++i) {
      const Ghost& g = rv[i];
      c->nbr[g.l * 4 + g.f] = int32_t(roff + int64_t(i));
      c->code[g.l * 4 + g.f] = uint8_t(32 + g.sface * 6 + g.sigma);
      c->recv_gid.push_back(g.sgid);
      c->recv_face.push_back(uint8_t(g.sface));
    }
    P.nrecv = int64_t(rv.size());
    roff += P.nrecv;
    auto& sv = sends[q];
    std::sort(sv.begin(), sv.end());
    for (auto& s : sv) {
      c->send_elem.push_back(int32_t(g2l[s.first]));
      c->send_face.push_back(uint8_t(s.second));
    }
    P.nsend = int64_t(sv.size());
    soff += P.nsend;
    c->peers.push_back(P);
  }
  c->nsend = soff;
  c->nrecv = roff;

  // ---- neighbour node tables (uint8) and face mask
  c->tbl.assign(96 * Nfp, 0);
  c->tblf.assign(96 * Nfp, 0);
  c->fmask8.assign(4 * Nfp, 0);
  for (int f = 0; f < 4; ++f) {
    for (int i = 0; i < Nfp; ++i) c->fmask8[f * Nfp + i] = uint8_t(c->ref.Fmask[f * Nfp + i]);
    for (int f2 = 0; f2 < 4; ++f2)
      for (int sg = 0; sg < 6; ++sg)
        for (int i = 0; i < Nfp; ++i) {
          int j = c->ref.nbr_local[((f * 4 + f2) * 6 + sg) * Nfp + i];
          c->tblf[(f * 24 + f2 * 6 + sg) * Nfp + i] = uint8_t(j);
          c->tbl[(f * 24 + f2 * 6 + sg) * Nfp + i] = uint8_t(c->ref.Fmask[f2 * Nfp + j]);
        }
  }

  // ---- modal scheme (reading A23): per face the ids of the tables that evaluate the own and
  // the neighbour polynomial at the face's integration points -- the points of the owner (the
  // smaller global id): t < 4 the standard points of face t, t = 4 + (f*4 + f2)*6 + perm the
  // points of face f carried onto face f2 of the neighbour (refelem.h ModalTables.Pmap)
  if (c->scheme == DG_SCHEME_MODAL) {
    static const int PERM_INV_H[6] = {0, 1, 2, 4, 3, 5};
    c->mtid.assign(size_t(c->K) * 8, 0);
    for (int64_t l = 0; l < c->K; ++l)
      for (int f = 0; f < 4; ++f) {
        const int code = c->code[l * 4 + f];
        int own = f, nbt = f;
        if (code < 32) {
          const int nb = c->nbr[l * 4 + f], f2 = code / 6, sg = code - 6 * f2;
          if (c->gid[l] < c->gid[nb]) {
            nbt = 4 + (f * 4 + f2) * 6 + sg;
          } else {
            own = 4 + (f2 * 4 + f) * 6 + PERM_INV_H[sg];
            nbt = f2;
          }
        }
        c->mtid[l * 8 + 2 * f] = uint8_t(own);
        c->mtid[l * 8 + 2 * f + 1] = uint8_t(nbt);
      }
  }

  // ---- DMMA B-fragment operator: Op = [-Dr -Ds -Dt 0 LIFT] (Np x KPAD), B[k][n] = Op[n][k];
  // the volume block is padded to a multiple of 4 columns (KVP) so the DMMA k-steps of
  // the volume and face halves of X never straddle (kernels.cuh Shape<N>)
  const int KV = 3 * Np, KVP = (KV + 3) / 4 * 4, KPAD = KVP + 4 * Nfp, NPAD = (Np + 7) / 8 * 8;
  const int KS4 = KPAD / 4, NTL = NPAD / 8;
  auto op = [&](int n, int k) -> double {
    if (n >= Np || k >= KPAD) return 0.0;
    if (k < Np) return -c->ref.Dr[n * Np + k];
    if (k < 2 * Np) return -c->ref.Ds[n * Np + k - Np];
    if (k < 3 * Np) return -c->ref.Dt[n * Np + k - 2 * Np];
    if (k < KVP) return 0.0;
    return c->ref.LIFT[n * 4 * Nfp + (k - KVP)];
  };
  // per k-step (OPW doubles, one contiguous block so the kernels can stream it in chunks):
  // NPG n-tile pairs of 64 doubles, lane l holding B(4ks+l%4, 8(2p)+l/4) and B(.., 8(2p+1)+l/4)
  // adjacent; then, for odd NTL, the trailing n-tile compacted to the lanes of its GS real
  // columns (l < 4 GS; for GS == 4 at N <= 4 transposed to [k = l % 4][column])
  const int NPG = NTL / 2, GS = (NTL % 2) ? Np - 8 * (NTL - 1) : 0, OPW = NPG * 64 + 4 * GS;
  const bool sbt = GS == 4 && N <= 4;
  c->opfrag.assign(size_t(KS4) * OPW, 0.0);
  for (int ks = 0; ks < KS4; ++ks) {
    double* o = c->opfrag.data() + size_t(ks) * OPW;
    for (int lane = 0; lane < 32; ++lane) {
      const int g = lane >> 2, t = lane & 3;
      for (int p = 0; p < NPG; ++p)
        for (int h = 0; h < 2; ++h) o[p * 64 + 2 * lane + h] = op(8 * (2 * p + h) + g, 4 * ks + t);
      // (GS == 4 in the warp-specialised kernel, N <= 4: stored [t][c], so a lane's four columns
      // are two adjacent 16-byte words)
      if (lane < 4 * GS) o[NPG * 64 + (sbt ? 4 * t + g : lane)] = op(8 * (NTL - 1) + g, 4 * ks + t);
    }
  }
  return DG_OK;
}

}  // namespace dgb
