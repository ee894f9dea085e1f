// sm_100a kernels of the nodal-DG Euler stage (Appendix A).
//
// One fused, persistent kernel per Runge-Kutta stage.  A CTA owns a tile of EB
// elements at a time:
//   A. TMA-free coalesced load of the tile's state Q[e][5][Np] and geometric
//      factors into shared memory;
//   B. pointwise volume flux (Eq. 1-2): contravariant fluxes
//      Ft_xi = xi_x F + xi_y G + xi_z H (xi = r,s,t) written row-major into the
//      shared operand X[(e,field)][k], k in [0, 3Np);
//   C. face traces: own trace from shared memory, neighbour trace gathered from
//      the neighbour's Q (vmapP encoded as neighbour element + face-permutation
//      code) or the halo buffer or a boundary ghost (wall: Eq. 4 mirror,
//      pass-through: Eq. 3, inflow: Eqs. 5-7), per-node wave speed, face max,
//      LLF flux, dF = Fscale (n.F(q-) - F*) written to X, k in [3Np, 3Np+4Nfp);
//   D. one dense contraction per tile on the FP64 tensor cores (DMMA,
//      mma.sync m16n8k4 f64):  rhs[(e,field)][n] = sum_k X[(e,field)][k] Op[n][k]
//      with Op = [-Dr -Ds -Dt LIFT] (Np x (3Np+4Nfp)) shared by every element,
//      held in shared memory in B-fragment order;
//   E. epilogue straight from the accumulator fragments: LSERK update
//      res = a res + dt rhs, Q_out = Q_in + b res (ping-pong Q, so neighbours of
//      later tiles still read the stage-input state), or rhs written out.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace dgk {

constexpr int GEO = 25;          // 9 metric terms + 4 faces x (nx, ny, nz, Fscale)
constexpr int CODE_GHOST = 32;   // 32 + f2*6 + sigma : neighbour trace in the halo buffer
constexpr int CODE_BC = 64;      // 64 + tag          : physical boundary

struct StageArgs {
  const double* Qin;      // [K][5][Np]
  double* Qout;           // [K][5][Np]   (MODE_UPDATE)
  double* res;            // [K][5][Np]   (MODE_UPDATE)
  double* out;            // [5][Kpub][Np] (MODE_RHS)
  const double* geo;      // [K][GEO]
  const int* nbr;         // [K][4]
  const uint8_t* code;    // [K][4]
  const int* pub;         // [K] public index
  const double* recv;     // [nrecv][5][Nfp]
  const double* op;       // B fragments
  const uint8_t* tbl;     // [4][4][6][Nfp] neighbour volume node  (local neighbours)
  const uint8_t* tblf;    // [4][4][6][Nfp] neighbour face-local node (halo records)
  const uint8_t* fmask;   // [4][Nfp]
  int* flag;              // [0] blow-up flag, [1] element id (global)
  const int64_t* gid;     // [K] global element id (for error messages)
  int e_begin, e_end;     // element range of this launch
  int Kpub;
  double gamma, a, b, dt, t;
  double pref;            // ambient pressure subtracted from the momentum fluxes (exact, A14)
  double qinf[5];
  double inflow_alpha;
  int lambda_mode;
};

template <int N>
struct Shape {
  static constexpr int NP = (N + 1) * (N + 2) * (N + 3) / 6;
  static constexpr int NFP = (N + 1) * (N + 2) / 2;
  static constexpr int KV = 3 * NP;
  static constexpr int KT = KV + 4 * NFP;
  static constexpr int KPAD = (KT + 3) / 4 * 4;
  static constexpr int KS4 = KPAD / 4;
  static constexpr int NPAD = (NP + 7) / 8 * 8;
  static constexpr int NTL = NPAD / 8;
  // row stride of X in doubles: >= KPAD and == 4 (mod 16) -> conflict-free A fragments
  static constexpr int XS = ((KPAD + 11) / 16) * 16 + 4;
  static constexpr int OPN = KS4 * NTL * 32;   // doubles in the B-fragment operator
};

template <int N>
struct Tile {
  // elements per tile; rows (element, field) padded to a multiple of 16 (the DMMA M)
  static constexpr int EB = (N <= 3) ? 32 : (N == 4 ? 16 : 8);
  static constexpr int NT = 512;
  static constexpr int ROWS = (5 * EB + 15) / 16 * 16;
  static constexpr int MT = ROWS / 16;
  static constexpr bool OP_SMEM = Shape<N>::OPN * 8 <= 72 * 1024;
  static constexpr int NTG = (Shape<N>::NTL >= 4) ? 2 : 1;          // n-tiles per work item
  static constexpr int NGRP = (Shape<N>::NTL + NTG - 1) / NTG;
  static constexpr int ITEMS = MT * NGRP;
  static constexpr size_t SMEM_X = size_t(ROWS) * Shape<N>::XS * 8;
  static constexpr size_t SMEM_OP = OP_SMEM ? size_t(Shape<N>::OPN) * 8 : 0;
  static constexpr size_t SMEM_Q = size_t(EB) * 5 * Shape<N>::NP * 8;
  static constexpr size_t SMEM_G = size_t(EB) * GEO * 8;
  static constexpr size_t SMEM_L = size_t(EB) * 4 * Shape<N>::NFP * 8;
  static constexpr size_t SMEM_T = size_t(2 * 96 * Shape<N>::NFP + 4 * Shape<N>::NFP + 15) / 16 * 16;
  static constexpr size_t SMEM = SMEM_X + SMEM_OP + SMEM_Q + SMEM_G + SMEM_L + SMEM_T;
  static_assert(SMEM <= 227 * 1024, "tile does not fit in shared memory");
};

__device__ __forceinline__ void dmma_16x8x4(double (&d)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

__device__ __forceinline__ void flag_blowup(int* flag, int64_t gid) {
  if (atomicCAS(flag, 0, 1) == 0) flag[1] = (int)gid;
}

// Eq. 5-7 inflow ghost (paper's scaled units), NEXT row N1
__device__ __forceinline__ void inflow_state(double t, double alpha, double gamma, double (&q)[5]) {
  double p = (t < 2.0 * M_PI / alpha) ? 1.0 + (0.05 - 0.05 * cos(alpha * t)) : 1.0;
  double rho = gamma * pow(p, 1.0 / gamma);
  double u = (p - 1.0) / (1.4 * 1.0);
  q[0] = rho;
  q[1] = rho * u;
  q[2] = 0.0;
  q[3] = 0.0;
  q[4] = p / (gamma - 1.0) + 0.5 * rho * u * u;
}

enum { MODE_UPDATE = 0, MODE_RHS = 1 };

template <int N, int MODE>
__global__ void __launch_bounds__(Tile<N>::NT, 1) stage_kernel(const StageArgs A) {
  using S = Shape<N>;
  using T = Tile<N>;
  constexpr int NP = S::NP, NFP = S::NFP, EB = T::EB, NT = T::NT, XS = S::XS;
  extern __shared__ __align__(16) unsigned char smem[];
  double* sX = reinterpret_cast<double*>(smem);
  double* sOp = sX + T::ROWS * XS;
  double* sQ = sOp + (T::OP_SMEM ? S::OPN : 0);
  double* sG = sQ + EB * 5 * NP;
  double* sL = sG + EB * GEO;
  uint8_t* sTbl = reinterpret_cast<uint8_t*>(sL + EB * 4 * NFP);
  uint8_t* sTblf = sTbl + 96 * NFP;
  uint8_t* sFm = sTblf + 96 * NFP;
  const int tid = threadIdx.x;
  const double* __restrict__ Op = T::OP_SMEM ? sOp : A.op;

  // one-time: operator, tables, zero the padding columns of X
  if (T::OP_SMEM)
    for (int i = tid; i < S::OPN; i += NT) sOp[i] = A.op[i];
  for (int i = tid; i < 96 * NFP; i += NT) {
    sTbl[i] = A.tbl[i];
    sTblf[i] = A.tblf[i];
  }
  for (int i = tid; i < 4 * NFP; i += NT) sFm[i] = A.fmask[i];
  for (int i = tid; i < T::ROWS * XS; i += NT) sX[i] = 0.0;   // padding rows/columns stay 0

  const double gamma = A.gamma, gm1 = A.gamma - 1.0;
  const int ntiles = (A.e_end - A.e_begin + EB - 1) / EB;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int e0 = A.e_begin + tile * EB;
    const int ne = min(EB, A.e_end - e0);
    __syncthreads();  // previous tile fully consumed
    // ---------------- A: load state + geometry (contiguous blocks)
    {
      const double* src = A.Qin + size_t(e0) * 5 * NP;
      const int n = ne * 5 * NP;
      for (int i = tid; i < n; i += NT) sQ[i] = __ldg(src + i);
      for (int i = n + tid; i < EB * 5 * NP; i += NT) sQ[i] = 0.0;
      const double* g = A.geo + size_t(e0) * GEO;
      for (int i = tid; i < ne * GEO; i += NT) sG[i] = __ldg(g + i);
    }
    __syncthreads();
    // ---------------- B: volume fluxes -> X[:, 0:3Np)
    for (int idx = tid; idx < EB * NP; idx += NT) {
      const int e = idx / NP, n = idx - e * NP;
      double* xr = sX + (e * 5) * XS;
      if (e >= ne) {
#pragma unroll
        for (int f = 0; f < 5; ++f) {
          xr[f * XS + n] = 0.0;
          xr[f * XS + NP + n] = 0.0;
          xr[f * XS + 2 * NP + n] = 0.0;
        }
        continue;
      }
      const double* q = sQ + e * 5 * NP + n;
      const double rho = q[0], mx = q[NP], my = q[2 * NP], mz = q[3 * NP], E = q[4 * NP];
      const double ri = 1.0 / rho;
      const double u = mx * ri, v = my * ri, w = mz * ri;
      const double p = gm1 * (E - 0.5 * (mx * u + my * v + mz * w));
      if (!(rho > 0.0) || !(p > 0.0) || !isfinite(E + mx + my + mz)) flag_blowup(A.flag, A.gid[e0 + e]);
      const double* G = sG + e * GEO;
      const double Ep = E + p;
      const double pd = p - A.pref;   // background-flux subtraction (A14)
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double cx = G[3 * d], cy = G[3 * d + 1], cz = G[3 * d + 2];
        // contravariant velocity and flux along xi_d
        const double U = cx * u + cy * v + cz * w;
        double* xc = xr + d * NP + n;
        xc[0] = rho * U;
        xc[XS] = mx * U + cx * pd;
        xc[2 * XS] = my * U + cy * pd;
        xc[3 * XS] = mz * U + cz * pd;
        xc[4 * XS] = Ep * U;
      }
    }
    // ---------------- C: face fluxes -> X[:, 3Np:3Np+4Nfp)
    constexpr int FN = EB * 4 * NFP;
    constexpr int FR = (FN + NT - 1) / NT;
    double qm[FR][5], qp[FR][5];
#pragma unroll
    for (int r = 0; r < FR; ++r) {
      const int idx = tid + r * NT;
      if (idx >= FN) continue;
      const int e = idx / (4 * NFP), fi = idx - e * 4 * NFP, f = fi / NFP, i = fi - f * NFP;
      if (e >= ne) {
        sL[idx] = 0.0;
        continue;
      }
      const int vm = sFm[fi];
      const double* q = sQ + e * 5 * NP + vm;
#pragma unroll
      for (int c = 0; c < 5; ++c) qm[r][c] = q[c * NP];
      const int ke = e0 + e;
      const int code = A.code[ke * 4 + f];
      const double* G = sG + e * GEO + 9 + 4 * f;
      const double nx = G[0], ny = G[1], nz = G[2];
      if (code < CODE_GHOST) {
        const int k2 = A.nbr[ke * 4 + f];
        const int node = sTbl[(f * 24 + code) * NFP + i];
        const double* q2 = A.Qin + size_t(k2) * 5 * NP + node;
#pragma unroll
        for (int c = 0; c < 5; ++c) qp[r][c] = __ldg(q2 + c * NP);
      } else if (code < CODE_BC) {
        const int g = A.nbr[ke * 4 + f];
        const int j = sTblf[(f * 24 + code - CODE_GHOST) * NFP + i];
        const double* q2 = A.recv + size_t(g) * 5 * NFP + j;
#pragma unroll
        for (int c = 0; c < 5; ++c) qp[r][c] = __ldg(q2 + c * NFP);
      } else {
        const int tag = code - CODE_BC;
        if (tag == 1) {  // reflective wall, Eq. 4 read as a mirror (A2)
          const double mn = qm[r][1] * nx + qm[r][2] * ny + qm[r][3] * nz;
          qp[r][0] = qm[r][0];
          qp[r][1] = qm[r][1] - 2.0 * mn * nx;
          qp[r][2] = qm[r][2] - 2.0 * mn * ny;
          qp[r][3] = qm[r][3] - 2.0 * mn * nz;
          qp[r][4] = qm[r][4];
        } else if (tag == 2) {  // pass-through: ambient state of Eq. 3
#pragma unroll
          for (int c = 0; c < 5; ++c) qp[r][c] = A.qinf[c];
        } else {  // inflow, Eqs. 5-7
          double qi[5];
          inflow_state(A.t, A.inflow_alpha, gamma, qi);
#pragma unroll
          for (int c = 0; c < 5; ++c) qp[r][c] = qi[c];
        }
      }
      // wave speeds |u.n| + c on both sides
      const double rim = 1.0 / qm[r][0], rip = 1.0 / qp[r][0];
      const double unm = (qm[r][1] * nx + qm[r][2] * ny + qm[r][3] * nz) * rim;
      const double unp = (qp[r][1] * nx + qp[r][2] * ny + qp[r][3] * nz) * rip;
      const double pm = gm1 * (qm[r][4] - 0.5 * (qm[r][1] * qm[r][1] + qm[r][2] * qm[r][2] + qm[r][3] * qm[r][3]) * rim);
      const double pp = gm1 * (qp[r][4] - 0.5 * (qp[r][1] * qp[r][1] + qp[r][2] * qp[r][2] + qp[r][3] * qp[r][3]) * rip);
      const double lm = fabs(unm) + sqrt(gamma * pm * rim);
      const double lp = fabs(unp) + sqrt(gamma * pp * rip);
      sL[idx] = fmax(lm, lp);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < FR; ++r) {
      const int idx = tid + r * NT;
      if (idx >= FN) continue;
      const int e = idx / (4 * NFP), fi = idx - e * 4 * NFP, f = fi / NFP;
      double* xd = sX + (e * 5) * XS + S::KV + fi;
      if (e >= ne) {
#pragma unroll
        for (int c = 0; c < 5; ++c) xd[c * XS] = 0.0;
        continue;
      }
      double lam;
      if (A.lambda_mode == 0) {
        const double* l = sL + e * 4 * NFP + f * NFP;
        lam = l[0];
#pragma unroll
        for (int j = 1; j < NFP; ++j) lam = fmax(lam, l[j]);
      } else {
        lam = sL[idx];
      }
      const double* G = sG + e * GEO + 9 + 4 * f;
      const double nx = G[0], ny = G[1], nz = G[2], fs = G[3];
      // normal fluxes n.F(q) on both sides
      double fm[5], fp[5];
      {
        const double ri = 1.0 / qm[r][0];
        const double un = (qm[r][1] * nx + qm[r][2] * ny + qm[r][3] * nz) * ri;
        const double p = gm1 * (qm[r][4] - 0.5 * (qm[r][1] * qm[r][1] + qm[r][2] * qm[r][2] + qm[r][3] * qm[r][3]) * ri);
        const double pd = p - A.pref;
        fm[0] = qm[r][0] * un;
        fm[1] = qm[r][1] * un + pd * nx;
        fm[2] = qm[r][2] * un + pd * ny;
        fm[3] = qm[r][3] * un + pd * nz;
        fm[4] = (qm[r][4] + p) * un;
      }
      {
        const double ri = 1.0 / qp[r][0];
        const double un = (qp[r][1] * nx + qp[r][2] * ny + qp[r][3] * nz) * ri;
        const double p = gm1 * (qp[r][4] - 0.5 * (qp[r][1] * qp[r][1] + qp[r][2] * qp[r][2] + qp[r][3] * qp[r][3]) * ri);
        const double pd = p - A.pref;
        fp[0] = qp[r][0] * un;
        fp[1] = qp[r][1] * un + pd * nx;
        fp[2] = qp[r][2] * un + pd * ny;
        fp[3] = qp[r][3] * un + pd * nz;
        fp[4] = (qp[r][4] + p) * un;
      }
      // dF = Fscale (n.F(q-) - F*),  F* = 1/2 (fm + fp) - 1/2 lam (q+ - q-)
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        const double fstar = 0.5 * (fm[c] + fp[c]) - 0.5 * lam * (qp[r][c] - qm[r][c]);
        xd[c * XS] = fs * (fm[c] - fstar);
      }
    }
    __syncthreads();
    // ---------------- D + E: DMMA contraction and epilogue
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
    for (int item = warp; item < T::ITEMS; item += NT / 32) {
      const int mt = item / T::NGRP, ng = item - mt * T::NGRP;
      double acc[T::NTG][4];
#pragma unroll
      for (int j = 0; j < T::NTG; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;
      const double* xa = sX + (mt * 16 + g) * XS + t4;
      const double* ob = Op + lane;
#pragma unroll 4
      for (int ks = 0; ks < S::KS4; ++ks) {
        const double a0 = xa[ks * 4], a1 = xa[8 * XS + ks * 4];
#pragma unroll
        for (int j = 0; j < T::NTG; ++j) {
          const int nt = ng * T::NTG + j;
          if (nt < S::NTL) dmma_16x8x4(acc[j], a0, a1, ob[(ks * S::NTL + nt) * 32]);
        }
      }
      // epilogue: rows (mt*16 + g, +8), cols nt*8 + 2*t4 + {0,1}
#pragma unroll
      for (int j = 0; j < T::NTG; ++j) {
        const int nt = ng * T::NTG + j;
        if (nt >= S::NTL) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = mt * 16 + g + 8 * h;
          const int e = row / 5, c = row - 5 * (row / 5);
          if (e >= ne) continue;
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int n = nt * 8 + 2 * t4 + q;
            if (n >= NP) continue;
            const double rhs = acc[j][2 * h + q];
            if (MODE == MODE_UPDATE) {
              const size_t gi = (size_t(e0 + e) * 5 + c) * NP + n;
              const double rr = A.a * A.res[gi] + A.dt * rhs;
              A.res[gi] = rr;
              A.Qout[gi] = sQ[(e * 5 + c) * NP + n] + A.b * rr;
            } else {
              A.out[(size_t(c) * A.Kpub + A.pub[e0 + e]) * NP + n] = rhs;
            }
          }
        }
      }
    }
  }
}

// pack the traces of this rank's partition faces: send[s][c][j] = Q[k][c][Fmask_f[j]]
template <int N>
__global__ void pack_kernel(const double* __restrict__ Q, const int* __restrict__ selem,
                            const uint8_t* __restrict__ sface, const uint8_t* __restrict__ fmask,
                            double* __restrict__ send, int64_t nrec) {
  constexpr int NP = Shape<N>::NP, NFP = Shape<N>::NFP;
  const int64_t total = nrec * 5 * NFP;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t s = i / (5 * NFP);
    const int rem = int(i - s * 5 * NFP), c = rem / NFP, j = rem - c * NFP;
    send[i] = Q[(size_t(selem[s]) * 5 + c) * NP + fmask[sface[s] * NFP + j]];
  }
}

// public [5][K][Np] <-> internal [K][5][Np]  (pub[k] = public index of internal element k)
__global__ void to_internal_kernel(const double* __restrict__ pubstate, const int* __restrict__ pub,
                                   double* __restrict__ Q, double* __restrict__ res, int64_t K, int Np) {
  const int64_t total = K * 5 * Np;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k = i / (5 * Np);
    const int rem = int(i - k * 5 * Np), c = rem / Np, n = rem - c * Np;
    Q[i] = pubstate[(size_t(c) * K + pub[k]) * Np + n];
    res[i] = 0.0;
  }
}

__global__ void to_public_kernel(const double* __restrict__ Q, const int* __restrict__ pub,
                                 double* __restrict__ pubstate, int64_t K, int Np) {
  const int64_t total = K * 5 * Np;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k = i / (5 * Np);
    const int rem = int(i - k * 5 * Np), c = rem / Np, n = rem - c * Np;
    pubstate[(size_t(c) * K + pub[k]) * Np + n] = Q[i];
  }
}

// per-block max of |u| + c over nodes (stable dt helper)
__global__ void max_speed_kernel(const double* __restrict__ Q, int64_t nnode, int Np, double gamma,
                                 double* __restrict__ partial) {
  __shared__ double red[32];
  double m = 0.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nnode; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k = i / Np;
    const int n = int(i - k * Np);
    const double* q = Q + size_t(k) * 5 * Np + n;
    const double rho = q[0], ri = 1.0 / rho;
    const double u = q[Np] * ri, v = q[2 * Np] * ri, w = q[3 * Np] * ri;
    const double p = (gamma - 1.0) * (q[4 * Np] - 0.5 * rho * (u * u + v * v + w * w));
    const double s = sqrt(u * u + v * v + w * w) + sqrt(gamma * p * ri);
    m = fmax(m, s);
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = (threadIdx.x < blockDim.x / 32) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) partial[blockIdx.x] = m;
  }
}

}  // namespace dgk
