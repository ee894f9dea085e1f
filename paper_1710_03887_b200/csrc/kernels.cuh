// sm_100a kernels of the nodal-DG Euler stage (Appendix A).
//
// One fused, persistent kernel per Runge-Kutta stage.  A CTA owns a tile of EB
// elements at a time:
//   A. load the tile's state Q[e][5][Np] and geometric factors into shared memory;
//   B. pointwise volume flux (Eq. 1-2): contravariant fluxes
//      Ft_xi = xi_x F + xi_y G + xi_z H (xi = r,s,t) written row-major into the
//      shared operand X[(e,field)][k], k in [0, 3Np);
//   C. face traces: own trace from shared memory, neighbour trace gathered from
//      the neighbour's Q (vmapP encoded as neighbour element + face-permutation
//      code) or the halo buffer or a boundary ghost (wall: Eq. 4 mirror,
//      pass-through: Eq. 3, inflow: Eqs. 5-7), per-node wave speed, face max,
//      LLF flux, dF = Fscale (n.F(q-) - F*) written to X, k in [KVP, KVP+4Nfp);
//   D. one dense contraction per tile on the FP64 tensor cores (DMMA,
//      mma.sync m16n8k4 f64):  rhs[(e,field)][n] = sum_k X[(e,field)][k] Op[n][k]
//      with Op = [-Dr -Ds -Dt 0 LIFT] (Np x KPAD) shared by every element, held
//      in shared memory in B-fragment order;
//   E. epilogue straight from the accumulator fragments: LSERK update
//      res = a res + dt rhs, Q_out = Q_in + b res (ping-pong Q, so neighbours of
//      later tiles still read the stage-input state), or rhs written out.
//
// stage_ws_kernel (N <= 4) is warp-specialised: 8 producer warps run A-C for
// tile i+1 while 8 consumer warps run D-E for tile i, handing over the volume
// and face halves of X through named barriers (bar.arrive / bar.sync).
// stage_kernel (N = 5, 6) runs A-E in lock-step with __syncthreads.
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
  static constexpr int KVP = (KV + 3) / 4 * 4;        // volume block padded to the DMMA k=4
  static constexpr int KPAD = KVP + 4 * NFP;          // face block starts at KVP
  static constexpr int KS4 = KPAD / 4;
  static constexpr int KSV = KVP / 4;                 // k-steps of the volume block
  static constexpr int NPAD = (NP + 7) / 8 * 8;
  static constexpr int NTL = NPAD / 8;
  // row stride of X in doubles: >= KPAD and == 12 (mod 16) -> conflict-free A fragments
  static constexpr int XS = (KPAD + 3) / 16 * 16 + 12;
  static constexpr int OPN = KS4 * NTL * 32;   // doubles in the B-fragment operator
};

__device__ __forceinline__ void dmma_16x8x4(double (&d)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }

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

// ---------------------------------------------------------------- pointwise pieces
// Volume flux at one node: q -> 15 contravariant flux values in X rows e*5+c, cols d*NP+n.
template <int NP, int XS>
__device__ __forceinline__ void volume_node(const double* q, const double* G, double* xr, double gm1, double pref,
                                            int* flag, int64_t gid) {
  const double rho = q[0], mx = q[NP], my = q[2 * NP], mz = q[3 * NP], E = q[4 * NP];
  const double ri = 1.0 / rho;
  const double u = mx * ri, v = my * ri, w = mz * ri;
  const double p = gm1 * (E - 0.5 * (mx * u + my * v + mz * w));
  if (!(rho > 0.0) || !(p > 0.0) || !isfinite(E + mx + my + mz)) flag_blowup(flag, gid);
  const double Ep = E + p;
  const double pd = p - pref;   // background-flux subtraction (A14)
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double cx = G[3 * d], cy = G[3 * d + 1], cz = G[3 * d + 2];
    const double U = cx * u + cy * v + cz * w;   // contravariant velocity along xi_d
    double* xc = xr + d * NP;
    xc[0] = rho * U;
    xc[XS] = fma(cx, pd, mx * U);
    xc[2 * XS] = fma(cy, pd, my * U);
    xc[3 * XS] = fma(cz, pd, mz * U);
    xc[4 * XS] = Ep * U;
  }
}

// Exterior trace q+ of face node i of face f: neighbour (local / halo) or boundary ghost.
template <int NP, int NFP>
__device__ __forceinline__ void exterior_trace(const StageArgs& A, int code, int nb, int f, int i, const uint8_t* tbl,
                                               const uint8_t* tblf, const double (&qm)[5], double nx, double ny,
                                               double nz, double (&qp)[5]) {
  if (code < CODE_GHOST) {
    const double* q2 = A.Qin + size_t(nb) * 5 * NP + tbl[(f * 24 + code) * NFP + i];
#pragma unroll
    for (int c = 0; c < 5; ++c) qp[c] = __ldg(q2 + c * NP);
  } else if (code < CODE_BC) {
    const double* q2 = A.recv + size_t(nb) * 5 * NFP + tblf[(f * 24 + code - CODE_GHOST) * NFP + i];
#pragma unroll
    for (int c = 0; c < 5; ++c) qp[c] = __ldg(q2 + c * NFP);
  } else {
    const int tag = code - CODE_BC;
    if (tag == 1) {  // reflective wall, Eq. 4 read as a mirror (A2)
      const double mn = qm[1] * nx + qm[2] * ny + qm[3] * nz;
      qp[0] = qm[0];
      qp[1] = qm[1] - 2.0 * mn * nx;
      qp[2] = qm[2] - 2.0 * mn * ny;
      qp[3] = qm[3] - 2.0 * mn * nz;
      qp[4] = qm[4];
    } else if (tag == 2) {  // pass-through: ambient state of Eq. 3
#pragma unroll
      for (int c = 0; c < 5; ++c) qp[c] = A.qinf[c];
    } else {  // inflow, Eqs. 5-7
      inflow_state(A.t, A.inflow_alpha, A.gamma, qp);
    }
  }
}

struct SideFlux {
  double f[5];   // n.F(q) with the ambient pressure subtracted (A14)
  double speed;  // |u.n| + c
};

__device__ __forceinline__ SideFlux side_flux(const double (&q)[5], double nx, double ny, double nz, double gamma,
                                              double pref) {
  SideFlux s;
  const double ri = 1.0 / q[0];
  const double un = (q[1] * nx + q[2] * ny + q[3] * nz) * ri;
  const double p = (gamma - 1.0) * (q[4] - 0.5 * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3]) * ri);
  const double pd = p - pref;
  s.f[0] = q[0] * un;
  s.f[1] = fma(pd, nx, q[1] * un);
  s.f[2] = fma(pd, ny, q[2] * un);
  s.f[3] = fma(pd, nz, q[3] * un);
  s.f[4] = (q[4] + p) * un;
  s.speed = fabs(un) + sqrt(gamma * p * ri);
  return s;
}

// ---------------------------------------------------------------- lock-step kernel (N = 5, 6)
template <int N>
struct Tile {
  static constexpr int EB = (N <= 3) ? 32 : (N == 4 ? 16 : 8);
  static constexpr int NT = 512;
  static constexpr int ROWS = (5 * EB + 15) / 16 * 16;
  static constexpr int MT = ROWS / 16;
  static constexpr bool OP_SMEM = Shape<N>::OPN * 8 <= 72 * 1024;
  static constexpr int NTG = (Shape<N>::NTL >= 4) ? 2 : 1;
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

template <int N, int MODE>
__global__ void __launch_bounds__(Tile<N>::NT, 1) stage_kernel(const StageArgs A) {
  using S = Shape<N>;
  using T = Tile<N>;
  constexpr int NP = S::NP, NFP = S::NFP, EB = T::EB, NT = T::NT, XS = S::XS;
  extern __shared__ __align__(128) unsigned char smem[];
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
    {
      const double* src = A.Qin + size_t(e0) * 5 * NP;
      const int n = ne * 5 * NP;
      for (int i = tid; i < n; i += NT) sQ[i] = __ldg(src + i);
      for (int i = n + tid; i < EB * 5 * NP; i += NT) sQ[i] = 0.0;
      const double* g = A.geo + size_t(e0) * GEO;
      for (int i = tid; i < ne * GEO; i += NT) sG[i] = __ldg(g + i);
    }
    __syncthreads();
    for (int idx = tid; idx < ne * NP; idx += NT) {
      const int e = idx / NP, n = idx - e * NP;
      volume_node<NP, XS>(sQ + e * 5 * NP + n, sG + e * GEO, sX + (e * 5) * XS + n, gm1, A.pref, A.flag, A.gid[e0 + e]);
    }
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
      const double* q = sQ + e * 5 * NP + sFm[fi];
#pragma unroll
      for (int c = 0; c < 5; ++c) qm[r][c] = q[c * NP];
      const int ke = e0 + e;
      const double* G = sG + e * GEO + 9 + 4 * f;
      exterior_trace<NP, NFP>(A, A.code[ke * 4 + f], A.nbr[ke * 4 + f], f, i, sTbl, sTblf, qm[r], G[0], G[1], G[2], qp[r]);
      const SideFlux sm = side_flux(qm[r], G[0], G[1], G[2], gamma, A.pref);
      const SideFlux sp = side_flux(qp[r], G[0], G[1], G[2], gamma, A.pref);
      sL[idx] = fmax(sm.speed, sp.speed);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < FR; ++r) {
      const int idx = tid + r * NT;
      if (idx >= FN) continue;
      const int e = idx / (4 * NFP), fi = idx - e * 4 * NFP, f = fi / NFP;
      double* xd = sX + (e * 5) * XS + S::KVP + fi;
      if (e >= ne) continue;
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
      const SideFlux sm = side_flux(qm[r], G[0], G[1], G[2], gamma, A.pref);
      const SideFlux sp = side_flux(qp[r], G[0], G[1], G[2], gamma, A.pref);
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        const double fstar = 0.5 * (sm.f[c] + sp.f[c]) - 0.5 * lam * (qp[r][c] - qm[r][c]);
        xd[c * XS] = G[3] * (sm.f[c] - fstar);
      }
    }
    __syncthreads();
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

// ---------------------------------------------------------------- warp-specialised kernel (N <= 4)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// TMA 1D bulk copy global -> shared, completion counted on an mbarrier (bytes % 16 == 0, 16B aligned)
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

template <int N>
struct WS {
  static constexpr int EB = (N <= 3) ? 32 : 16;
  static constexpr int PW = 8, CW = 8;                      // producer / consumer warps
  static constexpr int NT = 32 * (PW + CW);
  static constexpr int ROWS = 5 * EB;                       // multiple of 16
  static constexpr int MT = ROWS / 16;
  static_assert(ROWS % 16 == 0, "rows must fill DMMA m16 tiles");
  // consumer work items: (m-tile, group of NTG n-tiles); a consumer warp owns up to IPW items
  static constexpr int NTG = (Shape<N>::NTL >= 4) ? 2 : 1;
  static constexpr int NGRP = (Shape<N>::NTL + NTG - 1) / NTG;
  static constexpr int NTLP = NGRP * NTG;                   // n-tiles incl. a zero pad to fill groups
  static constexpr int ITEMS = MT * NGRP;
  static constexpr int IPW = (ITEMS + CW - 1) / CW;
  static constexpr int NSEG = 32 / Shape<N>::NFP;           // faces per producer warp-pass
  static constexpr int OPS = Shape<N>::KS4 * NTLP * 32;     // doubles of the grouped B operand
  // per-buffer bytes of the TMA-loaded tile inputs
  static constexpr uint32_t BQ = uint32_t(EB) * 5 * Shape<N>::NP * 8;
  static constexpr uint32_t BG = uint32_t(EB) * GEO * 8;
  static constexpr uint32_t BN = uint32_t(EB) * 4 * 4;
  static constexpr uint32_t BC = uint32_t(EB) * 4;
  static_assert(BQ % 16 == 0 && BG % 16 == 0 && BN % 16 == 0 && BC % 16 == 0, "TMA sizes");
  static constexpr size_t SMEM_X = size_t(ROWS) * Shape<N>::XS * 8;
  static constexpr size_t SMEM_OP = size_t(OPS) * 8;
  static constexpr size_t SMEM_IN = size_t(2) * (BQ + BG + BN + BC);
  static constexpr size_t SMEM_T = size_t(2 * 96 * Shape<N>::NFP + 4 * Shape<N>::NFP + 15) / 16 * 16;
  static constexpr size_t SMEM = SMEM_X + SMEM_OP + SMEM_IN + SMEM_T + 16;
  static_assert(SMEM <= 227 * 1024, "warp-specialised tile does not fit in shared memory");
  // named barriers
  static constexpr int BAR_P = 1, BAR_XV_FULL = 2, BAR_XV_EMPTY = 3, BAR_XF_FULL = 4, BAR_XF_EMPTY = 5, BAR_Q_EMPTY = 6;
};

template <int N, int MODE>
__global__ void __launch_bounds__(WS<N>::NT, 1) stage_ws_kernel(const StageArgs A) {
  using S = Shape<N>;
  using W = WS<N>;
  constexpr int NP = S::NP, NFP = S::NFP, EB = W::EB, XS = S::XS, NT = W::NT;
  constexpr int PT = 32 * W::PW;
  extern __shared__ __align__(128) unsigned char smem[];
  double* sX = reinterpret_cast<double*>(smem);
  double* sOp = sX + W::ROWS * XS;
  unsigned char* in0 = reinterpret_cast<unsigned char*>(sOp + W::OPS);
  // per buffer b: Q | geo | nbr | code
  auto bufQ = [&](int b) { return reinterpret_cast<double*>(in0 + b * (W::BQ + W::BG + W::BN + W::BC)); };
  auto bufG = [&](int b) { return reinterpret_cast<double*>(in0 + b * (W::BQ + W::BG + W::BN + W::BC) + W::BQ); };
  auto bufN = [&](int b) { return reinterpret_cast<int*>(in0 + b * (W::BQ + W::BG + W::BN + W::BC) + W::BQ + W::BG); };
  auto bufC = [&](int b) {
    return reinterpret_cast<uint8_t*>(in0 + b * (W::BQ + W::BG + W::BN + W::BC) + W::BQ + W::BG + W::BN);
  };
  uint8_t* sTbl = in0 + 2 * (W::BQ + W::BG + W::BN + W::BC);
  uint8_t* sTblf = sTbl + 96 * NFP;
  uint8_t* sFm = sTblf + 96 * NFP;
  uint64_t* sBar = reinterpret_cast<uint64_t*>(sTbl + W::SMEM_T);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // B operand regrouped per (k-step, n-tile group): lane reads its NTG values contiguously
  for (int i = tid; i < W::OPS; i += NT) {
    const int l = i % (32 * W::NTG), rest = i / (32 * W::NTG);
    const int grp = rest % W::NGRP, ks = rest / W::NGRP;
    const int ln = l / W::NTG, jj = l % W::NTG, nt = grp * W::NTG + jj;
    sOp[i] = nt < S::NTL ? A.op[(ks * S::NTL + nt) * 32 + ln] : 0.0;
  }
  for (int i = tid; i < 96 * NFP; i += NT) {
    sTbl[i] = A.tbl[i];
    sTblf[i] = A.tblf[i];
  }
  for (int i = tid; i < 4 * NFP; i += NT) sFm[i] = A.fmask[i];
  for (int i = tid; i < W::ROWS * XS; i += NT) sX[i] = 0.0;   // padding columns stay 0
  if (tid == 0) {
    mbar_init(&sBar[0], 1);
    mbar_init(&sBar[1], 1);
  }
  __syncthreads();

  const int ntiles = (A.e_end - A.e_begin + EB - 1) / EB;
  // tiles of this CTA: blockIdx.x, blockIdx.x + gridDim.x, ...
  const int nmine = (ntiles > (int)blockIdx.x) ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;

  if (warp < W::PW) {
    // ======================= producers: load (TMA), volume flux, face flux
    const double gamma = A.gamma, gm1 = A.gamma - 1.0;
    // inputs of local tile jj into buffer jj&1: TMA bulk copies for a full tile, plain loads otherwise
    auto fetch = [&](int jj) {
      const int tile = blockIdx.x + jj * gridDim.x;
      const int e0 = A.e_begin + tile * EB;
      const int ne = min(EB, A.e_end - e0);
      const int b = jj & 1;
      if (ne == EB) {
        if (tid == 0) {
          fence_proxy_async();
          mbar_arrive_expect_tx(&sBar[b], W::BQ + W::BG + W::BN + W::BC);
          tma_load_1d(bufQ(b), A.Qin + size_t(e0) * 5 * NP, W::BQ, &sBar[b]);
          tma_load_1d(bufG(b), A.geo + size_t(e0) * GEO, W::BG, &sBar[b]);
          tma_load_1d(bufN(b), A.nbr + size_t(e0) * 4, W::BN, &sBar[b]);
          tma_load_1d(bufC(b), A.code + size_t(e0) * 4, W::BC, &sBar[b]);
        }
      } else {
        double* q_s = bufQ(b);
        double* g_s = bufG(b);
        int* n_s = bufN(b);
        uint8_t* c_s = bufC(b);
        for (int i = tid; i < EB * 5 * NP; i += PT) q_s[i] = i < ne * 5 * NP ? __ldg(A.Qin + size_t(e0) * 5 * NP + i) : 0.0;
        for (int i = tid; i < EB * GEO; i += PT) g_s[i] = i < ne * GEO ? __ldg(A.geo + size_t(e0) * GEO + i) : 0.0;
        for (int i = tid; i < EB * 4; i += PT) {
          n_s[i] = i < ne * 4 ? __ldg(A.nbr + size_t(e0) * 4 + i) : 0;
          c_s[i] = i < ne * 4 ? A.code[size_t(e0) * 4 + i] : uint8_t(CODE_BC + 2);
        }
        nbar_sync(W::BAR_P, PT);
      }
    };
    if (nmine > 0) fetch(0);
    for (int j = 0; j < nmine; ++j) {
      const int tile = blockIdx.x + j * gridDim.x;
      const int e0 = A.e_begin + tile * EB;
      const int ne = min(EB, A.e_end - e0);
      const int buf = j & 1;
      const double* q_s = bufQ(buf);
      const double* g_s = bufG(buf);
      const int* n_s = bufN(buf);
      const uint8_t* c_s = bufC(buf);
      if (ne == EB) mbar_wait(&sBar[buf], (j >> 1) & 1);
      // ---- volume fluxes -> X[:, 0:3NP)
      if (j >= 1) nbar_sync(W::BAR_XV_EMPTY, NT);
      for (int idx = tid; idx < EB * NP; idx += PT) {
        const int e = idx / NP, n = idx - e * NP;
        double* xr = sX + (e * 5) * XS + n;
        if (e < ne) {
          volume_node<NP, XS>(q_s + e * 5 * NP + n, g_s + e * GEO, xr, gm1, A.pref, A.flag, A.gid[e0 + e]);
        } else {
#pragma unroll
          for (int c = 0; c < 5; ++c) {
            xr[c * XS] = 0.0;
            xr[c * XS + NP] = 0.0;
            xr[c * XS + 2 * NP] = 0.0;
          }
        }
      }
      nbar_arrive(W::BAR_XV_FULL, NT);
      // ---- prefetch the next tile's inputs (its buffer was last read by the epilogue of tile j-1)
      if (j + 1 < nmine) {
        if (j + 1 >= 2) nbar_sync(W::BAR_Q_EMPTY + ((j + 1) & 1), NT);
        fetch(j + 1);
      }
      // ---- face fluxes -> X[:, KVP:KVP+4NFP): one face per NFP-lane segment, two passes at a time
      if (j >= 1) nbar_sync(W::BAR_XF_EMPTY, NT);
      const int seg = lane / NFP, i = lane - seg * NFP;
      const bool lane_ok = seg < W::NSEG;
      constexpr int STRIDE = W::PW * W::NSEG;
      for (int fb = warp * W::NSEG; fb < EB * 4; fb += 2 * STRIDE) {
        double qm[2][5], qp[2][5], nv[2][4];
        bool act[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int face = fb + u * STRIDE + seg;
          const int e = face >> 2, f = face & 3;
          act[u] = lane_ok && face < EB * 4 && e < ne;
          if (act[u]) {
            const double* G = g_s + e * GEO + 9 + 4 * f;
            nv[u][0] = G[0]; nv[u][1] = G[1]; nv[u][2] = G[2]; nv[u][3] = G[3];
            const double* q = q_s + e * 5 * NP + sFm[f * NFP + i];
#pragma unroll
            for (int c = 0; c < 5; ++c) qm[u][c] = q[c * NP];
            exterior_trace<NP, NFP>(A, c_s[e * 4 + f], n_s[e * 4 + f], f, i, sTbl, sTblf, qm[u], nv[u][0], nv[u][1],
                                    nv[u][2], qp[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int face = fb + u * STRIDE + seg;
          const int e = face >> 2, f = face & 3;
          if (fb + u * STRIDE >= EB * 4) break;   // warp-uniform
          double lam = 0.0;
          SideFlux sm, sp;
          if (act[u]) {
            sm = side_flux(qm[u], nv[u][0], nv[u][1], nv[u][2], gamma, A.pref);
            sp = side_flux(qp[u], nv[u][0], nv[u][1], nv[u][2], gamma, A.pref);
            lam = fmax(sm.speed, sp.speed);
          }
          if (A.lambda_mode == 0) {
            // segmented max over the face's NFP lanes: inclusive scan, then broadcast the last
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
              const double o = __shfl_up_sync(0xffffffffu, lam, d);
              if (lane_ok && i >= d) lam = fmax(lam, o);
            }
            lam = __shfl_sync(0xffffffffu, lam, lane_ok ? seg * NFP + NFP - 1 : lane);
          }
          if (act[u]) {
            double* xd = sX + (e * 5) * XS + S::KVP + f * NFP + i;
#pragma unroll
            for (int c = 0; c < 5; ++c) {
              const double fstar = 0.5 * (sm.f[c] + sp.f[c]) - 0.5 * lam * (qp[u][c] - qm[u][c]);
              xd[c * XS] = nv[u][3] * (sm.f[c] - fstar);
            }
          } else if (lane_ok && face < EB * 4) {
            double* xd = sX + (e * 5) * XS + S::KVP + f * NFP + i;
#pragma unroll
            for (int c = 0; c < 5; ++c) xd[c * XS] = 0.0;
          }
        }
      }
      nbar_arrive(W::BAR_XF_FULL, NT);
    }
  } else {
    // ======================= consumers: DMMA contraction + LSERK epilogue
    const int cw = warp - W::PW, g = lane >> 2, t4 = lane & 3;
    int mt[W::IPW], ng[W::IPW];
    bool on[W::IPW];
#pragma unroll
    for (int it = 0; it < W::IPW; ++it) {
      const int item = cw + it * W::CW;
      on[it] = item < W::ITEMS;
      mt[it] = on[it] ? item / W::NGRP : 0;
      ng[it] = on[it] ? item - mt[it] * W::NGRP : 0;
    }
    for (int j = 0; j < nmine; ++j) {
      const int tile = blockIdx.x + j * gridDim.x;
      const int e0 = A.e_begin + tile * EB;
      const int ne = min(EB, A.e_end - e0);
      const int buf = j & 1;
      const double* q_s = bufQ(buf);
      double acc[W::IPW][W::NTG][4];
#pragma unroll
      for (int it = 0; it < W::IPW; ++it)
#pragma unroll
        for (int jj = 0; jj < W::NTG; ++jj) acc[it][jj][0] = acc[it][jj][1] = acc[it][jj][2] = acc[it][jj][3] = 0.0;
      auto kloop = [&](int k0, int k1) {
#pragma unroll 4
        for (int ks = k0; ks < k1; ++ks) {
#pragma unroll
          for (int it = 0; it < W::IPW; ++it) {
            if (!on[it]) continue;
            const double* xa = sX + (mt[it] * 16 + g) * XS + t4 + ks * 4;
            const double a0 = xa[0], a1 = xa[8 * XS];
            const double* ob = sOp + ((ks * W::NGRP + ng[it]) * 32 + lane) * W::NTG;
            if constexpr (W::NTG == 2) {
              const double2 b = *reinterpret_cast<const double2*>(ob);
              dmma_16x8x4(acc[it][0], a0, a1, b.x);
              dmma_16x8x4(acc[it][1], a0, a1, b.y);
            } else {
              dmma_16x8x4(acc[it][0], a0, a1, ob[0]);
            }
          }
        }
      };
      nbar_sync(W::BAR_XV_FULL, NT);
      kloop(0, S::KSV);
      if (j + 1 < nmine) nbar_arrive(W::BAR_XV_EMPTY, NT);
      // prefetch the residual while the face half of X is produced
      double rprev[W::IPW][W::NTG][4];
#pragma unroll
      for (int it = 0; it < W::IPW; ++it)
#pragma unroll
        for (int jj = 0; jj < W::NTG; ++jj)
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int row = mt[it] * 16 + g + 8 * h, e = row / 5, c = row - 5 * (row / 5);
              const int n = (ng[it] * W::NTG + jj) * 8 + 2 * t4 + q;
              const bool ok = MODE == MODE_UPDATE && on[it] && e < ne && n < NP;
              rprev[it][jj][2 * h + q] = ok ? __ldg(A.res + (size_t(e0 + e) * 5 + c) * NP + n) : 0.0;
            }
      nbar_sync(W::BAR_XF_FULL, NT);
      kloop(S::KSV, S::KS4);
      if (j + 1 < nmine) nbar_arrive(W::BAR_XF_EMPTY, NT);
#pragma unroll
      for (int it = 0; it < W::IPW; ++it) {
        if (!on[it]) continue;
#pragma unroll
        for (int jj = 0; jj < W::NTG; ++jj) {
          const int nt = ng[it] * W::NTG + jj;
          if (nt >= S::NTL) continue;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int row = mt[it] * 16 + g + 8 * h;
            const int e = row / 5, c = row - 5 * (row / 5);
            if (e >= ne) continue;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int n = nt * 8 + 2 * t4 + q;
              if (n >= NP) continue;
              const double rhs = acc[it][jj][2 * h + q];
              if (MODE == MODE_UPDATE) {
                const size_t gi = (size_t(e0 + e) * 5 + c) * NP + n;
                const double rr = fma(A.a, rprev[it][jj][2 * h + q], A.dt * rhs);
                A.res[gi] = rr;
                A.Qout[gi] = fma(A.b, rr, q_s[(e * 5 + c) * NP + n]);
              } else {
                A.out[(size_t(c) * A.Kpub + A.pub[e0 + e]) * NP + n] = rhs;
              }
            }
          }
        }
      }
      if (j + 2 < nmine) nbar_arrive(W::BAR_Q_EMPTY + buf, NT);
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
