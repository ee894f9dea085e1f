// Reference tetrahedron, library side.  See refelem.h.
//
// Nodes: warp & blend (Warburton 2006, blend parameter alpha = 0; DESIGN.md
// reading O1).  On the regular tetrahedron of edge 2 every edge (A,B)
// displaces a point by 4 lA lB w(lB - lA) (VB - VA)/2 with
//   w(x) = sum_{interior i} (xGLL_i - xEQ_i)/(1 - xEQ_i^2) prod_{interior j != i} (x - xEQ_j)/(xEQ_i - xEQ_j)
// (the 1D equispaced->Gauss-Lobatto displacement divided by the edge bubble);
// each face contributes its three edges blended by lb lc ld / prod(lx + la/2);
// points on tet edges take the 1D displacement.
//
// Operators: V_ij = psi_j(x_i) with psi the orthonormal PKDO
// polynomials; Dr = Vr V^-1; M^-1 = V V^T; face mass M_f = (V2 V2^T)^-1 with
// the orthonormal triangle basis in the face's parameter coordinates;
// LIFT = V V^T E.
#include "refelem.h"

#include <algorithm>
#include <cmath>
#include <string>

namespace dgb {

const int FACE_VERTS[4][3] = {{0, 1, 2}, {0, 1, 3}, {1, 2, 3}, {0, 2, 3}};
const int PERM6[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};

namespace {

// ---------------------------------------------------------------- Jacobi
// Orthonormal Jacobi polynomial P^(a,b)_n(x) (weight (1-x)^a (1+x)^b on [-1,1])
// by the three-term recurrence.
double jacobi(double x, double a, double b, int n) {
  double g0 = std::pow(2.0, a + b + 1) / (a + b + 1) * std::tgamma(a + 1) * std::tgamma(b + 1) /
              std::tgamma(a + b + 1);
  double p0 = 1.0 / std::sqrt(g0);
  if (n == 0) return p0;
  double g1 = (a + 1) * (b + 1) / (a + b + 3) * g0;
  double p1 = ((a + b + 2) * x / 2 + (a - b) / 2) / std::sqrt(g1);
  if (n == 1) return p1;
  double aold = 2.0 / (2 + a + b) * std::sqrt((a + 1) * (b + 1) / (a + b + 3));
  for (int i = 1; i < n; ++i) {
    double h1 = 2 * i + a + b;
    double anew = 2.0 / (h1 + 2) * std::sqrt((i + 1) * (i + 1 + a + b) * (i + 1 + a) * (i + 1 + b) / (h1 + 1) / (h1 + 3));
    double bnew = -(a * a - b * b) / h1 / (h1 + 2);
    double p2 = (-aold * p0 + (x - bnew) * p1) / anew;
    p0 = p1;
    p1 = p2;
    aold = anew;
  }
  return p1;
}

double djacobi(double x, double a, double b, int n) {
  if (n == 0) return 0.0;
  return std::sqrt(n * (n + a + b + 1)) * jacobi(x, a + 1, b + 1, n - 1);
}

// plain Legendre P_n and derivative (for the GLL points)
void legendre(int n, double x, double& p, double& dp) {
  double p0 = 1, p1 = x;
  if (n == 0) { p = 1; dp = 0; return; }
  for (int k = 1; k < n; ++k) {
    double p2 = ((2 * k + 1) * x * p1 - k * p0) / (k + 1);
    p0 = p1;
    p1 = p2;
  }
  p = p1;
  dp = n * (x * p1 - p0) / (x * x - 1);  // valid off +-1
}

std::vector<double> gll(int N) {
  std::vector<double> x(N + 1);
  x[0] = -1;
  x[N] = 1;
  for (int i = 1; i < N; ++i) {
    double z = -std::cos(M_PI * i / N);
    for (int it = 0; it < 100; ++it) {
      // roots of P_N'(x): Newton on q(x) = P_N'(x) using (1-x^2) P_N'' = 2x P_N' - N(N+1) P_N
      double p, dp;
      legendre(N, z, p, dp);
      double d2p = (2 * z * dp - N * (N + 1) * p) / (1 - z * z);
      double dz = dp / d2p;
      z -= dz;
      if (std::fabs(dz) < 1e-17) break;
    }
    x[i] = z;
  }
  std::sort(x.begin(), x.end());
  for (int i = 0; i <= N / 2; ++i) {  // symmetrise
    double m = 0.5 * (x[N - i] - x[i]);
    x[i] = -m;
    x[N - i] = m;
  }
  return x;
}

// ---------------------------------------------------------------- PKDO basis
// orthonormal tet basis psi_{ijk} and its (r,s,t) gradient (chain rule through
// the collapsed coordinates; every term is finite at the singular points)
void pkdo3(double r, double s, double t, int i, int j, int k, double& v, double& vr, double& vs, double& vt) {
  double a = (s + t != 0.0) ? 2 * (1 + r) / (-s - t) - 1 : -1.0;
  double b = (t != 1.0) ? 2 * (1 + s) / (1 - t) - 1 : -1.0;
  double c = t;
  double fa = jacobi(a, 0, 0, i), dfa = djacobi(a, 0, 0, i);
  double gb = jacobi(b, 2 * i + 1, 0, j), dgb = djacobi(b, 2 * i + 1, 0, j);
  double hc = jacobi(c, 2 * (i + j) + 2, 0, k), dhc = djacobi(c, 2 * (i + j) + 2, 0, k);
  const double C = 2.0 * std::sqrt(2.0);
  double omb = 1 - b, omc = 1 - c;
  v = C * fa * gb * std::pow(omb, i) * hc * std::pow(omc, i + j);
  // d/dr: fa' * 4/((1-b)(1-c)) * ...
  double tr = 0;
  if (i >= 1) tr = 4.0 * dfa * gb * std::pow(omb, i - 1) * hc * std::pow(omc, i + j - 1);
  // common "a-term" for s and t: fa' (1+a) 2/((1-b)(1-c)) gb (1-b)^i hc (1-c)^(i+j)
  double ta = 0;
  if (i >= 1) ta = 2.0 * dfa * (1 + a) * gb * std::pow(omb, i - 1) * hc * std::pow(omc, i + j - 1);
  // d/db [gb (1-b)^i]
  double dgb_full = dgb * std::pow(omb, i) - (i >= 1 ? i * gb * std::pow(omb, i - 1) : 0.0);
  double ts_b = 0, tt_b = 0;
  if (i + j >= 1) {
    double base = fa * dgb_full * hc * std::pow(omc, i + j - 1);
    ts_b = 2.0 * base;
    tt_b = (1 + b) * base;
  }
  // d/dc [hc (1-c)^(i+j)]
  double dhc_full = dhc * std::pow(omc, i + j) - (i + j >= 1 ? (i + j) * hc * std::pow(omc, i + j - 1) : 0.0);
  double tt_c = fa * gb * std::pow(omb, i) * dhc_full;
  vr = C * tr;
  vs = C * (ta + ts_b);
  vt = C * (ta + tt_b + tt_c);
}

// orthonormal triangle basis on {r,s >= -1, r+s <= 0} (area 2)
double pkdo2(double r, double s, int i, int j) {
  double a = (s != 1.0) ? 2 * (1 + r) / (1 - s) - 1 : -1.0;
  double b = s;
  return std::sqrt(2.0) * jacobi(a, 0, 0, i) * jacobi(b, 2 * i + 1, 0, j) * std::pow(1 - b, i);
}

// ---------------------------------------------------------------- dense LA
// In-place inverse by Gauss-Jordan with partial pivoting; n x n row-major.
bool invert(std::vector<double>& A, int n) {
  std::vector<double> I(n * n, 0.0);
  for (int i = 0; i < n; ++i) I[i * n + i] = 1;
  for (int c = 0; c < n; ++c) {
    int p = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(A[r * n + c]) > std::fabs(A[p * n + c])) p = r;
    if (A[p * n + c] == 0.0) return false;
    if (p != c)
      for (int k = 0; k < n; ++k) {
        std::swap(A[p * n + k], A[c * n + k]);
        std::swap(I[p * n + k], I[c * n + k]);
      }
    double d = A[c * n + c];
    for (int k = 0; k < n; ++k) {
      A[c * n + k] /= d;
      I[c * n + k] /= d;
    }
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      double f = A[r * n + c];
      if (f == 0.0) continue;
      for (int k = 0; k < n; ++k) {
        A[r * n + k] -= f * A[c * n + k];
        I[r * n + k] -= f * I[c * n + k];
      }
    }
  }
  A.swap(I);
  return true;
}

std::vector<double> matmul(const std::vector<double>& A, const std::vector<double>& B, int n, int m, int p) {
  std::vector<double> C(n * p, 0.0);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < m; ++k) {
      double a = A[i * m + k];
      for (int j = 0; j < p; ++j) C[i * p + j] += a * B[k * p + j];
    }
  return C;
}

}  // namespace

bool build_reference(int N, RefElem& R, std::string* msg) {
  R.N = N;
  R.Np = n_nodes(N);
  R.Nfp = n_face_nodes(N);
  const int Np = R.Np, Nfp = R.Nfp;

  // lattice (k outer, j, i inner) and integer barycentric weights (l1..l4)*N
  std::vector<int> lat;  // Np x 4
  for (int k = 0; k <= N; ++k)
    for (int j = 0; j <= N - k; ++j)
      for (int i = 0; i <= N - k - j; ++i) {
        lat.push_back(N - i - j - k);
        lat.push_back(i);
        lat.push_back(j);
        lat.push_back(k);
      }

  // ---- warp & blend on the regular tetrahedron of edge length 2
  const double s3 = std::sqrt(3.0), s6 = std::sqrt(6.0);
  const double VT[4][3] = {{-1, -1 / s3, -1 / s6}, {1, -1 / s3, -1 / s6}, {0, 2 / s3, -1 / s6}, {0, 0, 3 / s6}};
  std::vector<double> xg = gll(N);
  std::vector<double> xe(N + 1);
  for (int i = 0; i <= N; ++i) xe[i] = -1.0 + 2.0 * i / N;
  auto warp = [&](double x) {
    double w = 0;
    for (int i = 1; i < N; ++i) {
      double term = (xg[i] - xe[i]) / (1 - xe[i] * xe[i]);
      for (int j = 1; j < N; ++j)
        if (j != i) term *= (x - xe[j]) / (xe[i] - xe[j]);
      w += term;
    }
    return w;
  };
  // inverse of [VT^T; 1 1 1 1] for barycentric recovery
  std::vector<double> Bm(16);
  for (int v = 0; v < 4; ++v) {
    for (int d = 0; d < 3; ++d) Bm[d * 4 + v] = VT[v][d];
    Bm[12 + v] = 1.0;
  }
  if (!invert(Bm, 4)) { if (msg) *msg = "regular tet singular"; return false; }

  R.r.resize(Np); R.s.resize(Np); R.t.resize(Np);
  for (int n = 0; n < Np; ++n) {
    double lam[4];
    int nz = 0;
    for (int v = 0; v < 4; ++v) {
      lam[v] = double(lat[n * 4 + v]) / N;
      if (lat[n * 4 + v] == 0) ++nz;
    }
    double X[3] = {0, 0, 0}, sh[3] = {0, 0, 0};
    for (int d = 0; d < 3; ++d)
      for (int v = 0; v < 4; ++v) X[d] += lam[v] * VT[v][d];
    auto edge = [&](int a, int b, double wgt) {
      double amp = 4 * lam[a] * lam[b] * warp(lam[b] - lam[a]) * wgt;
      for (int d = 0; d < 3; ++d) sh[d] += amp * (VT[b][d] - VT[a][d]) / 2;
    };
    if (nz == 2) {
      int ab[2], c = 0;
      for (int v = 0; v < 4; ++v)
        if (lat[n * 4 + v] != 0) ab[c++] = v;
      edge(ab[0], ab[1], 1.0);
    } else if (nz < 2) {
      for (int f = 0; f < 4; ++f) {
        int b = FACE_VERTS[f][0], c = FACE_VERTS[f][1], d = FACE_VERTS[f][2];
        int a = 6 - b - c - d;
        double num = lam[b] * lam[c] * lam[d];
        if (num == 0.0) continue;
        double den = (lam[b] + lam[a] / 2) * (lam[c] + lam[a] / 2) * (lam[d] + lam[a] / 2);
        double blend = num / den;
        edge(b, c, blend);
        edge(c, d, blend);
        edge(b, d, blend);
      }
    }
    double Y[4] = {X[0] + sh[0], X[1] + sh[1], X[2] + sh[2], 1.0};
    double L[4];
    for (int v = 0; v < 4; ++v) {
      L[v] = 0;
      for (int q = 0; q < 4; ++q) L[v] += Bm[v * 4 + q] * Y[q];
    }
    R.r[n] = 2 * L[1] - 1;
    R.s[n] = 2 * L[2] - 1;
    R.t[n] = 2 * L[3] - 1;
  }

  // ---- face masks and face-local lattice coordinates
  R.Fmask.assign(4 * Nfp, 0);
  R.face_lat.assign(4 * Nfp * 3, 0);
  for (int f = 0; f < 4; ++f) {
    int opp = 6 - FACE_VERTS[f][0] - FACE_VERTS[f][1] - FACE_VERTS[f][2];
    int c = 0;
    for (int n = 0; n < Np; ++n)
      if (lat[n * 4 + opp] == 0) {
        if (c >= Nfp) { if (msg) *msg = "face node count"; return false; }
        R.Fmask[f * Nfp + c] = n;
        for (int m = 0; m < 3; ++m) R.face_lat[(f * Nfp + c) * 3 + m] = lat[n * 4 + FACE_VERTS[f][m]];
        ++c;
      }
    if (c != Nfp) { if (msg) *msg = "face node count"; return false; }
  }
  R.nbr_local.assign(4 * 4 * 6 * Nfp, -1);
  for (int f = 0; f < 4; ++f)
    for (int f2 = 0; f2 < 4; ++f2)
      for (int sg = 0; sg < 6; ++sg)
        for (int i = 0; i < Nfp; ++i) {
          int w2[3];
          for (int m = 0; m < 3; ++m) w2[PERM6[sg][m]] = R.face_lat[(f * Nfp + i) * 3 + m];
          int found = -1;
          for (int j = 0; j < Nfp; ++j) {
            const int* q = &R.face_lat[(f2 * Nfp + j) * 3];
            if (q[0] == w2[0] && q[1] == w2[1] && q[2] == w2[2]) { found = j; break; }
          }
          if (found < 0) { if (msg) *msg = "face permutation table"; return false; }
          R.nbr_local[((f * 4 + f2) * 6 + sg) * Nfp + i] = found;
        }

  // ---- Vandermonde matrices in the orthonormal basis
  std::vector<double> V(Np * Np), Vr(Np * Np), Vs(Np * Np), Vt(Np * Np);
  int m = 0;
  for (int i = 0; i <= N; ++i)
    for (int j = 0; j <= N - i; ++j)
      for (int k = 0; k <= N - i - j; ++k, ++m)
        for (int n = 0; n < Np; ++n)
          pkdo3(R.r[n], R.s[n], R.t[n], i, j, k, V[n * Np + m], Vr[n * Np + m], Vs[n * Np + m], Vt[n * Np + m]);
  std::vector<double> Vinv = V;
  if (!invert(Vinv, Np)) { if (msg) *msg = "singular Vandermonde"; return false; }
  R.Vinv = Vinv;
  R.Dr = matmul(Vr, Vinv, Np, Np, Np);
  R.Ds = matmul(Vs, Vinv, Np, Np, Np);
  R.Dt = matmul(Vt, Vinv, Np, Np, Np);

  // ---- LIFT = V V^T E
  std::vector<double> E(Np * 4 * Nfp, 0.0);
  for (int f = 0; f < 4; ++f) {
    std::vector<double> V2(Nfp * Nfp);
    for (int q = 0; q < Nfp; ++q) {
      int n = R.Fmask[f * Nfp + q];
      double a, b;  // face parameter coordinates
      if (f == 0) { a = R.r[n]; b = R.s[n]; }
      else if (f == 1) { a = R.r[n]; b = R.t[n]; }
      else { a = R.s[n]; b = R.t[n]; }
      int mm = 0;
      for (int i = 0; i <= N; ++i)
        for (int j = 0; j <= N - i; ++j, ++mm) V2[q * Nfp + mm] = pkdo2(a, b, i, j);
    }
    // M_f = (V2 V2^T)^-1
    std::vector<double> MM(Nfp * Nfp, 0.0);
    for (int p = 0; p < Nfp; ++p)
      for (int q = 0; q < Nfp; ++q) {
        double acc = 0;
        for (int l = 0; l < Nfp; ++l) acc += V2[p * Nfp + l] * V2[q * Nfp + l];
        MM[p * Nfp + q] = acc;
      }
    if (!invert(MM, Nfp)) { if (msg) *msg = "singular face Vandermonde"; return false; }
    for (int p = 0; p < Nfp; ++p)
      for (int q = 0; q < Nfp; ++q) E[R.Fmask[f * Nfp + p] * (4 * Nfp) + f * Nfp + q] = MM[p * Nfp + q];
  }
  std::vector<double> VVt(Np * Np, 0.0);
  for (int a = 0; a < Np; ++a)
    for (int b = 0; b < Np; ++b) {
      double acc = 0;
      for (int l = 0; l < Np; ++l) acc += V[a * Np + l] * V[b * Np + l];
      VVt[a * Np + b] = acc;
    }
  R.LIFT = matmul(VVt, E, Np, Np, 4 * Nfp);
  return true;
}

void interp_weights(const RefElem& R, double r, double s, double t, double* w) {
  const int N = R.N, Np = R.Np;
  std::vector<double> psi(Np);
  int m = 0;
  for (int i = 0; i <= N; ++i)
    for (int j = 0; j <= N - i; ++j)
      for (int k = 0; k <= N - i - j; ++k, ++m) {
        double dr, ds, dt;
        pkdo3(r, s, t, i, j, k, psi[m], dr, ds, dt);
      }
  for (int n = 0; n < Np; ++n) {
    double acc = 0;
    for (int j = 0; j < Np; ++j) acc += R.Vinv[j * Np + n] * psi[j];
    w[n] = acc;
  }
}

// ---------------------------------------------------------------- modal scheme (N3)
namespace {
// n-point Gauss-Jacobi rule for the weight (1-x)^alpha: Newton on the orthonormal Jacobi
// polynomial from Chebyshev guesses (with deflation), Christoffel weights 1/sum_k p_k(x)^2
void gauss_jacobi(int n, double alpha, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int k = 0; k < n; ++k) {
    double r = -std::cos((2.0 * k + 1) * M_PI / (2.0 * n));
    if (k > 0) r = 0.5 * (r + x[k - 1]);
    for (int it = 0; it < 200; ++it) {
      double f = jacobi(r, alpha, 0, n), df = djacobi(r, alpha, 0, n), s = 0;
      for (int i = 0; i < k; ++i) s += 1.0 / (r - x[i]);
      const double dr = f / (df - s * f);
      r -= dr;
      if (std::fabs(dr) < 1e-16) break;
    }
    x[k] = r;
  }
  std::sort(x.begin(), x.end());
  for (int k = 0; k < n; ++k) {
    double s = 0;
    for (int j = 0; j < n; ++j) {
      const double pj = jacobi(x[k], alpha, 0, j);
      s += pj * pj;
    }
    w[k] = 1.0 / s;
  }
}

void face_point(int f, double u, double v, double& r, double& s, double& t) {
  switch (f) {
    case 0: r = u; s = v; t = -1; break;
    case 1: r = u; s = -1; t = v; break;
    case 2: r = -1 - u - v; s = u; t = v; break;
    default: r = -1; s = u; t = v; break;
  }
}

const double REFV[4][3] = {{-1, -1, -1}, {1, -1, -1}, {-1, 1, -1}, {-1, -1, 1}};

void psi_row(const RefElem& R, double r, double s, double t, double* out, double* dr = nullptr, double* ds = nullptr,
             double* dt = nullptr) {
  int m = 0;
  for (int i = 0; i <= R.N; ++i)
    for (int j = 0; j <= R.N - i; ++j)
      for (int k = 0; k <= R.N - i - j; ++k, ++m) {
        double v, a, b, c;
        pkdo3(r, s, t, i, j, k, v, a, b, c);
        out[m] = v;
        if (dr) { dr[m] = a; ds[m] = b; dt[m] = c; }
      }
}
}  // namespace

const int PERM6_INV[6] = {0, 1, 2, 4, 3, 5};

bool build_modal(const RefElem& R, ModalTables& T, std::string* msg) {
  const int p = R.N, Np = R.Np, n = p + 1;
  T.p = p;
  T.Np = Np;
  std::vector<double> ga, wa, gb, wb, gc, wc;
  gauss_jacobi(n, 0, ga, wa);
  gauss_jacobi(n, 1, gb, wb);
  gauss_jacobi(n, 2, gc, wc);
  // orthonormal Jacobi weights integrate 1 to the weight's integral: check sum(wa) = 2
  double sa = 0;
  for (double v : wa) sa += v;
  if (std::fabs(sa - 2.0) > 1e-12) { if (msg) *msg = "Gauss-Jacobi rule"; return false; }
  T.NQ = n * n * n;
  T.NQF = n * n;
  T.wq.resize(T.NQ);
  T.Vq.assign(size_t(T.NQ) * Np, 0.0);
  T.Dq.assign(size_t(3) * Np * T.NQ, 0.0);
  std::vector<double> v(Np), dr(Np), ds(Np), dt(Np);
  int q = 0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      for (int k = 0; k < n; ++k, ++q) {
        const double a = ga[i], b = gb[j], c = gc[k];
        const double r = (1 + a) * (1 - b) * (1 - c) / 4 - 1, s = (1 + b) * (1 - c) / 2 - 1, t = c;
        T.wq[q] = wa[i] * wb[j] * wc[k] / 8;
        psi_row(R, r, s, t, v.data(), dr.data(), ds.data(), dt.data());
        for (int m = 0; m < Np; ++m) {
          T.Vq[size_t(q) * Np + m] = v[m];
          T.Dq[(size_t(0) * Np + m) * T.NQ + q] = T.wq[q] * dr[m];
          T.Dq[(size_t(1) * Np + m) * T.NQ + q] = T.wq[q] * ds[m];
          T.Dq[(size_t(2) * Np + m) * T.NQ + q] = T.wq[q] * dt[m];
        }
      }
  // face rule in the parameter (u, v), and the face barycentrics of its points
  std::vector<double> fu(T.NQF), fv(T.NQF);
  T.wf.resize(T.NQF);
  q = 0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j, ++q) {
      fu[q] = (1 + ga[i]) * (1 - gb[j]) / 2 - 1;
      fv[q] = gb[j];
      T.wf[q] = wa[i] * wb[j] / 2;
    }
  T.Pstd.assign(size_t(4) * T.NQF * Np, 0.0);
  T.Pmap.assign(size_t(96) * T.NQF * Np, 0.0);
  for (int fa = 0; fa < 4; ++fa)
    for (int qq = 0; qq < T.NQF; ++qq) {
      double r, s, t;
      face_point(fa, fu[qq], fv[qq], r, s, t);
      psi_row(R, r, s, t, &T.Pstd[(size_t(fa) * T.NQF + qq) * Np]);
      // barycentrics over the tet vertices, then over face fa's vertices
      const double lam[4] = {-(1 + r + s + t) / 2, (1 + r) / 2, (1 + s) / 2, (1 + t) / 2};
      double beta[3];
      for (int mm = 0; mm < 3; ++mm) beta[mm] = lam[FACE_VERTS[fa][mm]];
      for (int fb = 0; fb < 4; ++fb)
        for (int sg = 0; sg < 6; ++sg) {
          double x[3] = {0, 0, 0};
          for (int mm = 0; mm < 3; ++mm)
            for (int d = 0; d < 3; ++d) x[d] += beta[mm] * REFV[FACE_VERTS[fb][PERM6[sg][mm]]][d];
          psi_row(R, x[0], x[1], x[2], &T.Pmap[((size_t(fa * 4 + fb) * 6 + sg) * T.NQF + qq) * Np]);
        }
    }
  T.V.assign(size_t(Np) * Np, 0.0);
  for (int nn = 0; nn < Np; ++nn) psi_row(R, R.r[nn], R.s[nn], R.t[nn], &T.V[size_t(nn) * Np]);
  T.Vinv = R.Vinv;
  return true;
}

}  // namespace dgb
