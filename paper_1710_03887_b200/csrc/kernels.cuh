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
// tile i+1 while 4-8 consumer warps run D-E for tile i, handing over the volume
// and face halves of X through named barriers (bar.arrive / bar.sync).
// stage_ho_kernel (N = 5, 6) runs A-E in phases with all 16 warps and streams Op,
// too large to keep resident, through a TMA-fed shared-memory ring.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace dgk {

constexpr int GEO = 25;          // 9 metric terms + 4 faces x (nx, ny, nz, Fscale)
constexpr int CODE_GHOST = 32;   // 32 + f2*6 + sigma : neighbour trace in the halo buffer
constexpr int CODE_BC = 64;      // 64 + tag          : physical boundary
__device__ constexpr int PERM_INV[6] = {0, 1, 2, 4, 3, 5};   // inverse of the face-vertex permutations

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
  const double* op;       // B fragments (nodal) / concatenated modal tables (modal scheme)
  const uint8_t* tbl;     // [4][4][6][Nfp] neighbour volume node  (local neighbours)
  const uint8_t* tblf;    // [4][4][6][Nfp] neighbour face-local node (halo records)
  const uint8_t* fmask;   // [4][Nfp]
  const uint8_t* mtid;    // [K][4][2] modal face-point table ids (own, neighbour)
  int* flag;              // [0] blow-up flag, [1] element id (global)
  const int64_t* gid;     // [K] global element id (for error messages)
  int e_begin, e_end;     // element range of this launch
  int Kpub;
  double gamma, a, b, dt, t;
  double pref;            // ambient pressure subtracted from the momentum fluxes (exact, A14)
  double qinf[5];
  // inflow ghost (Eqs. 5-7; reading A24): ambient p0, rho0, c0 from q_inf
  // and gamma, pulse half amplitude in pressure units, angular frequency per scaled time unit
  double in_p0, in_rho0, in_c0, in_amp, in_omega;
  int lambda_mode;
  // timing experiments: 1 = skip the DMMA contraction, 2 = skip the flux arithmetic.  The host
  // passes the compile-time DG_DEBUG_SKIP (0 in product builds, no run-time switch); it is read
  // at run time because the N <= 4 kernels' measured schedules depend on those branches
  // (C4 54.3 vs 51.5 GDOF/s with the checks folded away)
  int skip;
  unsigned long long* trace;   // DG_TRACE builds: per-phase clock64 stamps of CTA 0
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

// Phase timestamps for one CTA (compiled in with -DDG_TRACE=1 only): slot = tile*16 + event.
#ifndef DG_TRACE
#define DG_TRACE 0
#endif
// Timing experiments only, compile time (tools/debug_sweep.sh builds with -DDG_DEBUG_SKIP=n):
// 1 = skip the DMMA contraction, 2 = skip the flux arithmetic.  Product builds: 0.
#ifndef DG_DEBUG_SKIP
#define DG_DEBUG_SKIP 0
#endif
#define DG_SKIPQ(x) (A.skip & (x))
__device__ __forceinline__ void trace_ev(const StageArgs& A, int j, int ev) {
  if (DG_TRACE && blockIdx.x == 0 && j < 64 && A.trace) {
    __syncwarp();
    unsigned long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
    if ((threadIdx.x & 31) == 0) A.trace[j * 16 + ev] = t;
  }
}

// per-warp stamps (DG_TRACE builds): slot 1024 + (tile*16 + warp)*8 + k (k < 8), tiles < 24
__device__ __forceinline__ void trace_w(const StageArgs& A, int j, int k) {
  if (DG_TRACE && blockIdx.x == 0 && j < 24 && A.trace) {
    __syncwarp();
    unsigned long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
    if ((threadIdx.x & 31) == 0) A.trace[1024 + (j * 16 + (threadIdx.x >> 5)) * 8 + k] = t;
  }
}

// rho > 0, p > 0 and all five conserved values finite, decided with integer ops on the
// IEEE bit patterns (keeps the check off the FP64 pipe)
__device__ __forceinline__ bool state_ok(double rho, double p, double mx, double my, double mz, double E) {
  const long long r = __double_as_longlong(rho), pp = __double_as_longlong(p);
  const long long EXP = 0x7ff0000000000000LL;
  const bool fin = ((__double_as_longlong(mx) & EXP) != EXP) & ((__double_as_longlong(my) & EXP) != EXP) &
                   ((__double_as_longlong(mz) & EXP) != EXP) & ((__double_as_longlong(E) & EXP) != EXP);
  // positive, non-zero, finite (NaN and +inf have the exponent all ones)
  const bool rpos = (r > 0) & ((r & EXP) != EXP);
  const bool ppos = (pp > 0) & ((pp & EXP) != EXP);
  return fin & rpos & ppos;
}

__device__ __forceinline__ void flag_blowup(int* flag, int64_t gid) {
  if (atomicCAS(flag, 0, 1) == 0) flag[1] = (int)gid;
}

// Eqs. 5-7 inflow ghost (NEXT row N1; reading A24):
//   p = p0 + (a - a cos(omega t)) for omega t < 2 pi, else p0      (scaled p0 = 1, a = 0.05)
//   rho = rho0 (p / p0)^(1/gamma)                                   (Eq. 6, C = gamma at rho0 = 1.4, p0 = 1)
//   u = (p - p0) / (rho0 c0),  v = w = 0                            (Eq. 5)
//   E = p / (gamma - 1) + rho u^2 / 2                               (Eq. 7)
__device__ __forceinline__ void inflow_state(const StageArgs& A, double (&q)[5]) {
  const double wt = A.in_omega * A.t;
  const double p = (wt < 2.0 * M_PI) ? A.in_p0 + (A.in_amp - A.in_amp * cos(wt)) : A.in_p0;
  const double rho = A.in_rho0 * pow(p / A.in_p0, 1.0 / A.gamma);
  const double u = (p - A.in_p0) / (A.in_rho0 * A.in_c0);
  q[0] = rho;
  q[1] = rho * u;
  q[2] = 0.0;
  q[3] = 0.0;
  q[4] = p / (A.gamma - 1.0) + 0.5 * rho * u * u;
}

enum { MODE_UPDATE = 0, MODE_RHS = 1 };

// Programmatic dependent launch of the stage kernels (bit N of DG_PDL: order N; default N = 1-4):
// a stage's CTA may start on an SM as soon as the previous stage's CTA there has exited and run
// its prologue (operator, tables, barriers, ghost states) while other SMs finish; it waits for
// the whole previous grid (griddepcontrol.wait) before touching the state.  Hides the launch
// latency and the prologue between the five stage launches of a step: C2 (44 us per stage) 55.1
// -> 56.3 GDOF/s, C1 2.3 -> 2.7, C4 56.0 -> 56.2.
#ifndef DG_PDL
#define DG_PDL 30
#endif
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// Reciprocal and square root from the MUFU seeds plus one third-order correction each
// (seed error e -> O(e^3), below 1 ulp for the ~2^-20 seeds): within ~1 ulp of the
// correctly rounded results (the parity tests bound the effect), at a fraction of the
// issue cost of IEEE div/sqrt with their slow-path branches.
//   1/x:     e = 1 - x y,   y' = y (1 + e + e^2)                  (x y' = 1 - e^3)
//   sqrt(x): d = 1 - x y^2, sqrt(x) = x y (1 - d)^(-1/2) = x y (1 + d/2 + 3 d^2/8 + O(d^3))
#ifndef DG_NEWTON2
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;\n" : "=d"(y) : "d"(x));
  const double e = fma(-x, y, 1.0);
  return fma(y, fma(e, e, e), y);
}
__device__ __forceinline__ double sqrt_nr(double x) {   // x > 0
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;\n" : "=d"(y) : "d"(x));
  const double xy = x * y;
  const double d = fma(-xy, y, 1.0);
  return fma(xy, d * fma(0.375, d, 0.5), xy);
}
#else   // two Newton steps each (the previous form; experiment knob)
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;\n" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
__device__ __forceinline__ double sqrt_nr(double x) {   // x > 0
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;\n" : "=d"(y) : "d"(x));
  double e = fma(-x * y, y, 1.0);
  y = fma(0.5 * y, e, y);
  e = fma(-x * y, y, 1.0);
  y = fma(0.5 * y, e, y);
  return x * y;
}
#endif

// Neighbour trace for a paired face (local element or halo record); boundary faces are filled later.
template <int NP, int NFP>
__device__ __forceinline__ void gather_trace(const StageArgs& A, int code, int nb, int f, int i, const uint8_t* tbl,
                                             const uint8_t* tblf, double (&qp)[5]) {
  if (code < CODE_GHOST) {
    const double* q2 = A.Qin + size_t(nb) * 5 * NP + tbl[(f * 24 + code) * NFP + i];
#pragma unroll
    for (int c = 0; c < 5; ++c) qp[c] = __ldg(q2 + c * NP);
  } else if (code < CODE_BC) {
    const double* q2 = A.recv + size_t(nb) * 5 * NFP + tblf[(f * 24 + code - CODE_GHOST) * NFP + i];
#pragma unroll
    for (int c = 0; c < 5; ++c) qp[c] = __ldg(q2 + c * NFP);
  }
}

// Boundary ghost of face node with interior trace qm (wall: Eq. 4 mirror, pass-through: Eq. 3, inflow: Eqs. 5-7).
__device__ __forceinline__ void ghost_trace(const StageArgs& A, int tag, const double (&qm)[5], double nx, double ny,
                                            double nz, double (&qp)[5]) {
  if (tag == 1) {
    const double mn = qm[1] * nx + qm[2] * ny + qm[3] * nz;
    qp[0] = qm[0];
    qp[1] = qm[1] - 2.0 * mn * nx;
    qp[2] = qm[2] - 2.0 * mn * ny;
    qp[3] = qm[3] - 2.0 * mn * nz;
    qp[4] = qm[4];
  } else if (tag == 2) {
#pragma unroll
    for (int c = 0; c < 5; ++c) qp[c] = A.qinf[c];
  } else {
    inflow_state(A, qp);
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

__device__ __forceinline__ void tma_store_1d(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_store_commit_and_wait_read() {
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}

template <int XSTR_, int K0_, int K1_>
struct KBlk {   // k-steps [K0, K1) of the X block that starts at k-step K0
  static constexpr int XSTR = XSTR_, K0 = K0_, K1 = K1_;
};

// Neighbour traces of NPASS face passes (face of pass u: fbase + u fstride; one face per
// SEGW-lane segment, lane i < NFP its node i): local neighbour / halo record gathers, or the
// boundary ghost from the own trace; idle lanes keep a finite filler.
template <int N, int NPASS>
__device__ __forceinline__ void face_gather(const StageArgs& A, int fbase, int fstride, int flim, int ne, int i,
                                            bool lane_ok, const double* q_s, const double* g_s, const int* n_s,
                                            const uint8_t* c_s, const uint8_t* sTbl, const uint8_t* sTblf,
                                            const uint8_t* sFm, double (&qp)[NPASS][5]) {
  constexpr int NP = Shape<N>::NP, NFP = Shape<N>::NFP;
  // DG_GATHER2 (default: N = 3 and N = 1; C3 61.7 -> 64.1, C2 52.0 -> 53.2 GDOF/s; at N = 4 55.6 ->
  // 52.4; at N = 2 with 12 + 4 warps 55.2 vs 57.9 without)
#ifndef DG_GATHER2
#define DG_GATHER2 1
#endif
  if constexpr (DG_GATHER2 == 2 || (DG_GATHER2 == 1 && (N == 3 || N == 1))) {
    // all passes' shared-memory lookups level by level (code and neighbour, then the node
    // table), so the passes' dependent load chains overlap instead of running one after another
    int code[NPASS], nb[NPASS], node[NPASS];
    bool ok[NPASS];
#pragma unroll
    for (int u = 0; u < NPASS; ++u) {
      const int face = fbase + u * fstride;
      const int e = face >> 2, f = face & 3;
      ok[u] = !DG_SKIPQ(2) && lane_ok && face < flim && e < ne;
      const int ec = ok[u] ? e : 0;
      code[u] = ok[u] ? int(c_s[ec * 4 + f]) : CODE_BC;
      nb[u] = n_s[ec * 4 + f];
    }
#pragma unroll
    for (int u = 0; u < NPASS; ++u) {
      const int f = (fbase + u * fstride) & 3;
      const int ii = lane_ok ? i : 0;
      node[u] = code[u] < CODE_GHOST ? int(sTbl[(f * 24 + code[u]) * NFP + ii])
                : code[u] < CODE_BC ? int(sTblf[(f * 24 + code[u] - CODE_GHOST) * NFP + ii]) : int(sFm[f * NFP + ii]);
    }
#pragma unroll
    for (int u = 0; u < NPASS; ++u) {
#pragma unroll
      for (int c = 0; c < 5; ++c) qp[u][c] = A.qinf[c];
      if (code[u] < CODE_GHOST) {
        const double* q2 = A.Qin + size_t(nb[u]) * 5 * NP + node[u];
#pragma unroll
        for (int c = 0; c < 5; ++c) qp[u][c] = __ldg(q2 + c * NP);
      } else if (code[u] < CODE_BC) {
        const double* q2 = A.recv + size_t(nb[u]) * 5 * NFP + node[u];
#pragma unroll
        for (int c = 0; c < 5; ++c) qp[u][c] = __ldg(q2 + c * NFP);
      } else if (ok[u]) {   // boundary ghost from the own trace (Q of this tile is in shared memory)
        const int face = fbase + u * fstride;
        const int e = face >> 2, f = face & 3;
        const double* G = g_s + e * GEO + 9 + 4 * f;
        const double* q = q_s + e * 5 * NP + node[u];
        double qm[5];
#pragma unroll
        for (int c = 0; c < 5; ++c) qm[c] = q[c * NP];
        ghost_trace(A, code[u] - CODE_BC, qm, G[0], G[1], G[2], qp[u]);
      }
    }
  } else {
#pragma unroll
  for (int u = 0; u < NPASS; ++u) {
    const int face = fbase + u * fstride;
    const int e = face >> 2, f = face & 3;
#pragma unroll
    for (int c = 0; c < 5; ++c) qp[u][c] = A.qinf[c];
    if (!DG_SKIPQ(2) && lane_ok && face < flim && e < ne) {
      const int code = c_s[e * 4 + f];
      if (code < CODE_BC) {
        gather_trace<NP, NFP>(A, code, n_s[e * 4 + f], f, i, sTbl, sTblf, qp[u]);
      } else {   // boundary ghost from the own trace (Q of this tile is in shared memory)
        const double* G = g_s + e * GEO + 9 + 4 * f;
        const double* q = q_s + e * 5 * NP + sFm[f * NFP + i];
        double qm[5];
#pragma unroll
        for (int c = 0; c < 5; ++c) qm[c] = q[c * NP];
        ghost_trace(A, code - CODE_BC, qm, G[0], G[1], G[2], qp[u]);
      }
    }
  }
  }
}

// Face terms of NPASS passes into the face block of X (row stride XSF, column f Nfp + i):
// stage 1 both sides' primitives and node speeds (passes as independent chains), stage 2 the
// face max by an xor butterfly within the SEGW-lane segment (integer pipe: positive doubles
// order like their bit patterns, idle lanes hold 0), stage 3
//   Fscale (n.F(q-) - F*) = Fscale/2 ((n.F(q-) - n.F(q+)) + lam (q+ - q-)),
// where the ambient-pressure shift (A14) cancels in n.F(q-) - n.F(q+).  Slots of elements past
// ne store zeros.
template <int N, int NPASS, int SEGW, int XSF>
__device__ __forceinline__ void face_terms(const StageArgs& A, int fbase, int fstride, int flim, int ne, int i,
                                           bool lane_ok, const double* q_s, const double* g_s, const uint8_t* sFm,
                                           const double (&qp)[NPASS][5], double* sXf) {
  constexpr int NP = Shape<N>::NP, NFP = Shape<N>::NFP;
  if DG_SKIPQ(2) return;
  const double gamma = A.gamma, gm1 = A.gamma - 1.0;
  // DG_F1 (default): the own trace is read from shared memory once -- the first pass keeps
  // q+ - q- and n.F(q-) - n.F(q+) (10 values per pass, as many as the primitives it replaced),
  // the second pass only applies the face max
#ifndef DG_F1
#define DG_F1 2
#endif
  // (N = 4: 8 B of spills, still C4 54.3 -> 55.7 GDOF/s; C3 59.6 -> 60.3)
  constexpr bool F1 = DG_F1 == 2 || (DG_F1 == 1 && N <= 3);
  double rip[NPASS], unp[NPASS], pp[NPASS], lam[NPASS], unmv[NPASS], pmv[NPASS];
  double dqv[F1 ? NPASS : 1][5], gfv[F1 ? NPASS : 1][5];
#pragma unroll
  for (int u = 0; u < NPASS; ++u) {
    const int face = fbase + u * fstride;
    const bool act = lane_ok && face < flim && (face >> 2) < ne;
    const int fc = act ? face : 0;
    const int e = fc >> 2, f = fc & 3, ii = lane_ok ? i : 0;
    const double* G = g_s + e * GEO + 9 + 4 * f;
    const double nx = G[0], ny = G[1], nz = G[2];
    const double* q = q_s + e * 5 * NP + sFm[f * NFP + ii];
    const double qm0 = q[0], qm1 = q[NP], qm2 = q[2 * NP], qm3 = q[3 * NP], qm4 = q[4 * NP];
    const double rim = rcp_nr(qm0);
    const double unm = (qm1 * nx + qm2 * ny + qm3 * nz) * rim;
    const double pm = gm1 * (qm4 - 0.5 * (qm1 * qm1 + qm2 * qm2 + qm3 * qm3) * rim);
    unmv[u] = unm;
    pmv[u] = pm;
    rip[u] = rcp_nr(qp[u][0]);
    unp[u] = (qp[u][1] * nx + qp[u][2] * ny + qp[u][3] * nz) * rip[u];
    pp[u] = gm1 * (qp[u][4] - 0.5 * (qp[u][1] * qp[u][1] + qp[u][2] * qp[u][2] + qp[u][3] * qp[u][3]) * rip[u]);
    const double l = fmax(fabs(unm) + sqrt_nr(gamma * pm * rim), fabs(unp[u]) + sqrt_nr(gamma * pp[u] * rip[u]));
    lam[u] = act ? l : 0.0;
    if constexpr (F1) {
      const double dp = pm - pp[u];
      gfv[u][0] = fma(qm0, unm, -qp[u][0] * unp[u]);
      gfv[u][1] = fma(dp, nx, fma(qm1, unm, -qp[u][1] * unp[u]));
      gfv[u][2] = fma(dp, ny, fma(qm2, unm, -qp[u][2] * unp[u]));
      gfv[u][3] = fma(dp, nz, fma(qm3, unm, -qp[u][3] * unp[u]));
      gfv[u][4] = fma(qm4 + pm, unm, -(qp[u][4] + pp[u]) * unp[u]);
      dqv[u][0] = qp[u][0] - qm0;
      dqv[u][1] = qp[u][1] - qm1;
      dqv[u][2] = qp[u][2] - qm2;
      dqv[u][3] = qp[u][3] - qm3;
      dqv[u][4] = qp[u][4] - qm4;
    }
  }
  if (A.lambda_mode == 0) {
    if constexpr ((SEGW & (SEGW - 1)) == 0) {
#pragma unroll
      for (int d = 1; d < SEGW; d <<= 1) {
#pragma unroll
        for (int u = 0; u < NPASS; ++u) {
          const long long a = __double_as_longlong(lam[u]);
          const long long o = __shfl_xor_sync(0xffffffffu, a, d);
          lam[u] = __longlong_as_double(a > o ? a : o);
        }
      }
    } else {
      // segments of SEGW = Nfp lanes (not a power of two): cyclic rotations within the segment,
      // the window doubling each step (1, 2, 4, 8 ... >= Nfp); lanes outside a segment read themselves
      const int lane = threadIdx.x & 31;
      const int sb = lane - i;
#pragma unroll
      for (int d = 1; d < SEGW; d <<= 1) {
        const int src = lane_ok ? sb + (i + d) % SEGW : lane;
#pragma unroll
        for (int u = 0; u < NPASS; ++u) {
          const long long a = __double_as_longlong(lam[u]);
          const long long o = __shfl_sync(0xffffffffu, a, src);
          lam[u] = __longlong_as_double(a > o ? a : o);
        }
      }
    }
  }
  if constexpr (F1) {
#pragma unroll
    for (int u = 0; u < NPASS; ++u) {
      const int face = fbase + u * fstride;
      const bool slot = lane_ok && face < flim;
      const bool act = slot && (face >> 2) < ne;
      const int fc = slot ? face : 0;
      const int e = fc >> 2, f = fc & 3, ii = lane_ok ? i : 0;
      const double hfs = act ? 0.5 * g_s[e * GEO + 9 + 4 * f + 3] : 0.0;
      double* xd = sXf + (e * 5) * XSF + f * NFP + ii;
      if (slot) {
#pragma unroll
        for (int c = 0; c < 5; ++c) xd[c * XSF] = act ? hfs * fma(lam[u], dqv[u][c], gfv[u][c]) : 0.0;
      }
    }
  } else {
#pragma unroll
  for (int u = 0; u < NPASS; ++u) {
    const int face = fbase + u * fstride;
    const bool slot = lane_ok && face < flim;
    const bool act = slot && (face >> 2) < ne;
    const int fc = slot ? face : 0;
    const int e = fc >> 2, f = fc & 3, ii = lane_ok ? i : 0;
    const double* G = g_s + e * GEO + 9 + 4 * f;
    const double nx = G[0], ny = G[1], nz = G[2], hfs = act ? 0.5 * G[3] : 0.0;
    const double* q = q_s + e * 5 * NP + sFm[f * NFP + ii];
    double qm[5];
#pragma unroll
    for (int c = 0; c < 5; ++c) qm[c] = q[c * NP];
    const double pm = pmv[u], unm = unmv[u], dp = pm - pp[u];
    double df[5];
    df[0] = fma(qm[0], unm, -qp[u][0] * unp[u]);
    df[1] = fma(dp, nx, fma(qm[1], unm, -qp[u][1] * unp[u]));
    df[2] = fma(dp, ny, fma(qm[2], unm, -qp[u][2] * unp[u]));
    df[3] = fma(dp, nz, fma(qm[3], unm, -qp[u][3] * unp[u]));
    df[4] = fma(qm[4] + pm, unm, -(qp[u][4] + pp[u]) * unp[u]);
    double* xd = sXf + (e * 5) * XSF + f * NFP + ii;
    if (slot) {
#pragma unroll
      for (int c = 0; c < 5; ++c) xd[c * XSF] = act ? hfs * fma(lam[u], qp[u][c] - qm[c], df[c]) : 0.0;
    }
  }
  }
}

// Pointwise volume flux of node slot idx of a tile (Eq. 1-2): contravariant fluxes
// Ft_d = xi_d,x F + xi_d,y G + xi_d,z H (d = r, s, t) into the volume block of X, row (e, field),
// column d Np + n; slots past the tile's nodes compute on a clamped node and store zeros (or
// nothing past the tile), so the loop around it can stay branch-free.
template <int N, int XSV>
__device__ __forceinline__ void vol_node(const StageArgs& A, int idx, const double* q_s, const double* g_s, int e0,
                                         int ne, double gm1, double* sXv, int ebn) {
  constexpr int NP = Shape<N>::NP;
  const bool inb = idx < ebn;
  const int ic = inb ? idx : 0;
  const int e = ic / NP, n = ic - e * NP;
  const bool act = inb && e < ne;
  const double* q = q_s + e * 5 * NP + n;
  const double rho = q[0], mx = q[NP], my = q[2 * NP], mz = q[3 * NP], E = q[4 * NP];
  const double ri = rcp_nr(rho);
  const double u = mx * ri, v = my * ri, w = mz * ri;
  const double p = gm1 * (E - 0.5 * (mx * u + my * v + mz * w));
  if (act && !state_ok(rho, p, mx, my, mz, E)) flag_blowup(A.flag, A.gid[e0 + e]);
  const double* G = g_s + e * GEO;
  const double Ep = E + p, pd = p - A.pref;   // background-flux subtraction (A14)
  double f[3][5];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double cx = G[3 * d], cy = G[3 * d + 1], cz = G[3 * d + 2];
    const double U = cx * u + cy * v + cz * w;   // contravariant velocity along xi_d
    f[d][0] = rho * U;
    f[d][1] = fma(cx, pd, mx * U);
    f[d][2] = fma(cy, pd, my * U);
    f[d][3] = fma(cz, pd, mz * U);
    f[d][4] = Ep * U;
  }
  if (inb) {
    double* xr = sXv + (e * 5) * XSV + n;
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int c = 0; c < 5; ++c) xr[c * XSV + d * NP] = act ? f[d][c] : 0.0;
  }
}

// V: tile variant (N = 2 only: V = 1 is the 32-element tile for small meshes, where the 48-element
// default leaves SMs without a tile)
template <int N, int V = 0>
struct WS {
#ifndef DG_WS_EB2
#define DG_WS_EB2 48
#endif
#ifdef DG_WS_EB
  static constexpr int EB = DG_WS_EB;
#else
  static constexpr int EB = N == 2 ? (V == 1 ? 32 : DG_WS_EB2) : N == 1 ? 32 : 16;
#endif
  // producer / consumer warps (DG_WS_PW / DG_WS_CW override for experiments); at N = 2, 3 the
  // flux work is the larger share, so 12 producer and 4 consumer warps (measured on C3; N = 2 on
  // the C4 mesh: a third of the stall samples were consumers waiting for X, 52.5 -> 54.2 GDOF/s,
  // 57.9 with the plain face gathers)
#ifdef DG_WS_PW
  static constexpr int PW = DG_WS_PW;
#else
  static constexpr int PW = (N == 3 || N == 2) ? 12 : 8;
#endif
#ifdef DG_WS_CW
  static constexpr int CW = DG_WS_CW;
#else
  static constexpr int CW = (N == 3 || N == 2) ? 4 : 8;
#endif
  static constexpr int NT = 32 * (PW + CW);
  static constexpr int PT = 32 * PW, CT = 32 * CW;
  static constexpr int ROWS = 5 * EB;                       // multiple of 8 (DMMA m8 row tiles)
  static_assert(ROWS % 8 == 0, "rows must fill DMMA m8 tiles");
  // faces per producer warp-pass: one face per power-of-two lane segment (butterfly face max)
  // N = 3: dense segments of Nfp = 10 lanes (3 faces per warp pass, 2 passes instead of 3 with
  // 16-lane segments: a third fewer face-term instructions); face max by rotations
#ifndef DG_FDENSE
#define DG_FDENSE 1
#endif
  static constexpr bool FDENSE = DG_FDENSE && N == 3;
  static constexpr int SEGW = FDENSE ? Shape<N>::NFP
                              : Shape<N>::NFP <= 4 ? 4 : Shape<N>::NFP <= 8 ? 8 : Shape<N>::NFP <= 16 ? 16 : 32;
  static constexpr int NSEG = 32 / SEGW;
  static constexpr int FPASS = (4 * EB + PW * NSEG - 1) / (PW * NSEG);   // face passes per producer warp
  // X is split into its volume block [ROWS][XSV] and face block [ROWS][XSF];
  // strides == 12 (mod 16) doubles keep the A-fragment loads conflict-free
  // when Np == 4 (mod 16) (N = 1, 3), XSV == 4 (mod 16) also makes consecutive elements' volume
  // rows continue each other's bank sequence (5 XSV == Np mod 16): conflict-free flux stores
#ifndef DG_XSV4
#define DG_XSV4 1
#endif
  static constexpr bool XS4 = DG_XSV4 && Shape<N>::NP % 16 == 4;
  static constexpr int XSV = XS4 ? (Shape<N>::KVP + 11) / 16 * 16 + 4 : (Shape<N>::KVP + 3) / 16 * 16 + 12;
  static constexpr int XSF = (4 * Shape<N>::NFP + 3) / 16 * 16 + 12;
  // B operand in shared memory, per k-step: NPG n-tile pairs (64 doubles, a lane's two values
  // adjacent) then, if NTL is odd, the trailing n-tile compacted to the lanes of its GS real
  // columns (lane = 4 g + t, g < GS)
  static constexpr int NPG = Shape<N>::NTL / 2, HS = Shape<N>::NTL % 2;
  static constexpr int GS = HS ? Shape<N>::NP - 8 * (Shape<N>::NTL - 1) : 0;
  static constexpr int OPW = NPG * 64 + 4 * GS;
  static constexpr int OPC = Shape<N>::KS4 * OPW;
  // per-buffer bytes of the TMA-loaded tile inputs
  static constexpr uint32_t BQ = uint32_t(EB) * 5 * Shape<N>::NP * 8;
  static constexpr uint32_t BG = uint32_t(EB) * GEO * 8;
  static constexpr uint32_t BN = uint32_t(EB) * 4 * 4;
  static constexpr uint32_t BC = uint32_t(EB) * 4;
  static constexpr uint32_t BIN = BQ + BG + BN + BC;
  static_assert(BQ % 16 == 0 && BG % 16 == 0 && BN % 16 == 0 && BC % 16 == 0, "TMA sizes");
  static constexpr size_t SMEM_XV = size_t(ROWS) * XSV * 8;
  static constexpr size_t SMEM_XF = size_t(ROWS) * XSF * 8;
  static constexpr size_t SMEM_OP = (size_t(OPC) * 8 + 15) / 16 * 16;
  // input buffers (Q, geometry, connectivity) and residual tiles: 3 and 2 when they fit (the
  // producers then never wait for the consumers' epilogue, the residual arrives a tile early),
  // else 2 and 1
  static constexpr size_t SMEM_T = size_t(2 * 96 * Shape<N>::NFP + 4 * Shape<N>::NFP + 15) / 16 * 16;
  static constexpr bool DEEP = SMEM_XV + SMEM_XF + SMEM_OP + SMEM_T + 64 + 3 * size_t(BIN) + 2 * size_t(BQ) <= 227 * 1024;
  static constexpr int NIN = DEEP ? 3 : 2, NRES = DEEP ? 2 : 1;
  static constexpr size_t SMEM_IN = size_t(NIN) * BIN;
  static constexpr size_t SMEM_RES = size_t(NRES) * BQ;                  // residual tiles (TMA in/out)
  static constexpr size_t SMEM = SMEM_XV + SMEM_XF + SMEM_OP + SMEM_IN + SMEM_RES + SMEM_T + 64;
  static_assert(SMEM <= 227 * 1024, "warp-specialised tile does not fit in shared memory");
  // named barriers
  static constexpr int BAR_P = 1, BAR_XV_FULL = 2, BAR_XV_EMPTY = 3, BAR_XF_FULL = 4, BAR_XF_EMPTY = 5,
                       BAR_Q_EMPTY = 6 /* .. 6 + NIN - 1 */, BAR_C = 9;
};

// consumer k-loop unroll (register pressure vs load hoisting): measured best 7 at N = 4
// (C4 55.1 vs 54.9 GDOF/s at 6), 6 at N <= 3; DG_KUNROLL overrides for experiments
template <int N>
constexpr int kunroll() {
#ifdef DG_KUNROLL
  return DG_KUNROLL;
#else
  return N == 4 ? 7 : N == 3 ? 15 : 6;   // N = 3: both loops (15 and 10 k-steps) fully unrolled (C3 64.8 -> 65.7)
#endif
}

template <int N, int MODE, int V = 0>
struct ConsumerIO {
  const StageArgs& A;
  double* sXv;
  double* sXf;
  const double* sOp;
  unsigned char* in0;
  double* sRes;
  uint64_t* barRes;
  uint64_t* barIn;
  int nmine, ctid, lane;
};

__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a0, double b0) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a0), "d"(b0));
}

// Balanced work split for the consumers: units are (8-row tile, n-tile pair) and (8-row tile,
// odd trailing n-tile).  Pairs go round-robin over the consumer warps; singles are placed one at
// a time on the warp minimising (its SMSP's load, its own load) -- warp cw runs on SMSP cw % 4 --
// in FP64-pipe cycles per k-step: a pair 32 (two DMMA), a single 2 GS on DFMA (16 as a DMMA),
// plus, for a warp's first single, DG_SBV (the per-k-step B loads of the odd tile, which every
// warp holding singles repeats; 4 by default, so singles gather on few warps).  The plan is a
// compile-time constant every consumer thread reads.
#ifndef DG_SBV
#define DG_SBV 0
#endif
template <int N, int V = 0>
struct M8Plan {
  static constexpr int MT8 = WS<N, V>::ROWS / 8;
  static constexpr int NPG = WS<N, V>::NPG, HS = WS<N, V>::HS;
  static constexpr int P = MT8 * NPG, SG = MT8 * HS, CW = WS<N, V>::CW;
  static constexpr int CPMAX = (P + CW - 1) / CW;
  static constexpr bool SDF1 = WS<N, V>::GS > 0 && WS<N, V>::GS <= 4;
#ifdef DG_SWSI
  static constexpr int WSI = DG_SWSI;
#else
  static constexpr int WSI = 16;   // pipe-exact 2 GS concentrates singles: C3 56.9 vs 61.8 GDOF/s
#endif
  static constexpr int SBV = P > 0 ? DG_SBV : 0;   // singles only (N = 1): spread them
  struct Owners {
    int w[SG > 0 ? SG : 1];
  };
  static constexpr Owners owners() {
    Owners o{};
    int load[CW] = {}, smsp[4] = {}, ns[CW] = {};
    for (int w = 0; w < CW; ++w) {
      load[w] = 32 * (P > w ? (P - 1 - w) / CW + 1 : 0);
      smsp[w % 4] += load[w];
    }
    for (int s = 0; s < SG; ++s) {
      int best = 0;
      for (int w = 1; w < CW; ++w) {
        const int cb = WSI + (ns[best] ? 0 : SBV), cc = WSI + (ns[w] ? 0 : SBV);
        // with a B-load term, ties go to a warp that already loads the odd tile's B values
        const int a = ((smsp[w % 4] + cc) * 4096 + load[w] + cc) * 2 + (SBV > 0 && ns[w] == 0);
        const int b = ((smsp[best % 4] + cb) * 4096 + load[best] + cb) * 2 + (SBV > 0 && ns[best] == 0);
        if (a < b) best = w;
      }
      const int c = WSI + (ns[best] ? 0 : SBV);
      load[best] += c;
      smsp[best % 4] += c;
      ++ns[best];
      o.w[s] = best;
    }
    return o;
  }
  static constexpr int count(int w) {
    int n = 0;
    for (int s = 0; s < SG; ++s) n += owners().w[s] == w;
    return n;
  }
  static constexpr int maxcount() {
    int m = 0;
    for (int w = 0; w < CW; ++w) m = count(w) > m ? count(w) : m;
    return m;
  }
  static constexpr int CSMAX = maxcount() > 0 ? maxcount() : 1;
  static constexpr int npairs(int w) { return P > w ? (P - 1 - w) / CW + 1 : 0; }
  static constexpr bool occurs(int pa, int si) {
    for (int w = 0; w < CW; ++w)
      if (npairs(w) == pa && count(w) == si) return true;
    return false;
  }
};

template <int N, int V = 0>
__device__ __forceinline__ void m8_singles(int cw, int* out, int& count) {
  using PL = M8Plan<N, V>;
  constexpr typename PL::Owners o = PL::owners();
  count = 0;
#pragma unroll
  for (int s = 0; s < PL::SG; ++s)
    if (o.w[s] == cw) out[count++] = s;
}

// Consumer warp: DMMA m8n8k4 over its units, then the LSERK epilogue.  Full tiles run the
// epilogue in shared memory: the residual tile arrives by TMA (issued one tile ahead), res and
// Q are updated in place and leave by two TMA bulk stores.  Partial tiles and MODE_RHS use
// plain global accesses.
template <int N, int MODE, int NPAIR, int NSING, int V = 0>
__device__ __forceinline__ void ws_consumer_m8(const ConsumerIO<N, MODE, V>& io, int cw, const int* singles) {
  using S = Shape<N>;
  using W = WS<N, V>;
  using PL = M8Plan<N, V>;
  constexpr int NP = S::NP, EB = W::EB, NT = W::NT, XSV = W::XSV, XSF = W::XSF;
  const StageArgs& A = io.A;
  const int lane = io.lane, g = lane >> 2, t4 = lane & 3;
  int mtp[NPAIR > 0 ? NPAIR : 1], ntp[NPAIR > 0 ? NPAIR : 1], mts[NSING > 0 ? NSING : 1];
#pragma unroll
  for (int k = 0; k < NPAIR; ++k) {
    const int p = cw + k * W::CW;
    constexpr int NPG1 = PL::NPG > 0 ? PL::NPG : 1;
    mtp[k] = p / NPG1;
    ntp[k] = 2 * (p % NPG1);
  }
#pragma unroll
  for (int k = 0; k < NSING; ++k) mts[k] = singles[k];
  constexpr int NSLOT = 2 * NPAIR + NSING;
  // the consumer warp whose lane 0 issues the tile's TMA traffic (residual load, input refill,
  // bulk stores) and waits for the bulk-store reads: the last one (fewest pair units; measured
  // C4 55.0 vs 54.9, C3 55.0 vs 54.8 GDOF/s with warp 0)
#ifdef DG_WS_IOW
  constexpr int IOW = DG_WS_IOW < W::CW ? DG_WS_IOW : 0;
#else
  constexpr int IOW = W::CW - 1;
#endif
  constexpr int IOT = 32 * IOW;
  // IODEFER: the IO thread does not wait for a tile's bulk-store reads at the end of its
  // epilogue; the input refill / release and (NRES == 1) the residual load follow at the next
  // tile's XV_FULL
#ifdef DG_IODEFER
  constexpr bool IODEFER = DG_IODEFER;
#else
  constexpr bool IODEFER = N == 3;   // C3 66.0 -> 66.3 GDOF/s; at N = 4 (producers the bound) 56.0 -> 54.6
#endif
  auto tile_full = [&](int jj) {
    const int e0 = A.e_begin + (int(blockIdx.x) + jj * int(gridDim.x)) * EB;
    return A.e_end - e0 >= EB;
  };
  auto res_buf = [&](int jj) { return io.sRes + (jj % W::NRES) * (W::BQ / 8); };
  auto load_res = [&](int jj) {   // one thread; the last bulk store from that buffer has been read
    const int e0 = A.e_begin + (int(blockIdx.x) + jj * int(gridDim.x)) * EB;
    fence_proxy_async();
    mbar_arrive_expect_tx(io.barRes + jj % W::NRES, W::BQ);
    tma_load_1d(res_buf(jj), A.res + size_t(e0) * 5 * NP, W::BQ, io.barRes + jj % W::NRES);
  };
  // with two input buffers the consumer that releases a buffer (its Q bulk store has been read)
  // refills it with the inputs of the tile two ahead, so the producers never wait for it
  auto fetch_in = [&](int jj) {   // one thread, full tiles only
    const int e0 = A.e_begin + (int(blockIdx.x) + jj * int(gridDim.x)) * EB;
    const int b = jj % W::NIN;
    unsigned char* ib = io.in0 + b * W::BIN;
    fence_proxy_async();
    mbar_arrive_expect_tx(io.barIn + b, W::BIN);
    tma_load_1d(ib, A.Qin + size_t(e0) * 5 * NP, W::BQ, io.barIn + b);
    tma_load_1d(ib + W::BQ, A.geo + size_t(e0) * GEO, W::BG, io.barIn + b);
    tma_load_1d(ib + W::BQ + W::BG, A.nbr + size_t(e0) * 4, W::BN, io.barIn + b);
    tma_load_1d(ib + W::BQ + W::BG + W::BN, A.code + size_t(e0) * 4, W::BC, io.barIn + b);
  };
  if (MODE == MODE_UPDATE && io.ctid == IOT && io.nmine > 0 && tile_full(0)) load_res(0);
  for (int j = 0; j < io.nmine; ++j) {
    const int tile = blockIdx.x + j * gridDim.x;
    const int e0 = A.e_begin + tile * EB;
    const int ne = min(EB, A.e_end - e0);
    const int buf = j % W::NIN;
    double* q_s = reinterpret_cast<double*>(io.in0 + buf * W::BIN);
    double* sRes = res_buf(j);
    double acc[NSLOT > 0 ? NSLOT : 1][2];
#pragma unroll
    for (int u = 0; u < NSLOT; ++u) acc[u][0] = acc[u][1] = 0.0;
    // the odd n-tile has only GS real columns: with GS <= 4 it is cheaper on DFMA (GS per k-step
    // and lane, partial sums over the lane's k = t mod 4, reduced by two shuffles) than as a
    // full 8-column DMMA (16 pipe cycles for GS useful columns)
#ifndef DG_SDF
#define DG_SDF 1
#endif
    constexpr bool SDF = DG_SDF && W::GS > 0 && W::GS <= 4;
    double sacc[NSING > 0 ? NSING : 1][4];
#pragma unroll
    for (int k = 0; k < NSING; ++k) sacc[k][0] = sacc[k][1] = sacc[k][2] = sacc[k][3] = 0.0;
    auto unit_mt = [&](int u) { return u < 2 * NPAIR ? mtp[u >> 1] : mts[u - 2 * NPAIR]; };
    auto unit_nt = [&](int u) { return u < 2 * NPAIR ? ntp[u >> 1] + (u & 1) : S::NTL - 1; };
    // output column of accumulator (u, q): DMMA fragment layout, or (SDF singles) column t of
    // the odd n-tile in slot q = 0
    auto unit_n = [&](int u, int q) {
      if (SDF && u >= 2 * NPAIR) return q == 0 ? (S::NTL - 1) * 8 + t4 : NP;
      return unit_nt(u) * 8 + 2 * t4 + q;
    };
    auto kloop = [&](auto xblk) {
      constexpr int XSTR = decltype(xblk)::XSTR, K0 = decltype(xblk)::K0, K1 = decltype(xblk)::K1;
      if DG_SKIPQ(1) return;
      const double* X = (K0 == 0) ? io.sXv : io.sXf;
      constexpr int KU = kunroll<N>();
#pragma unroll KU
      for (int ks = K0; ks < K1; ++ks) {
        const double* ob = io.sOp + ks * W::OPW;
#pragma unroll
        for (int k = 0; k < NPAIR; ++k) {
          const double a0 = X[(mtp[k] * 8 + g) * XSTR + t4 + (ks - K0) * 4];
          const double2 b = *reinterpret_cast<const double2*>(ob + (ntp[k] >> 1) * 64 + 2 * lane);
          dmma_8x8x4(acc[2 * k], a0, b.x);
          dmma_8x8x4(acc[2 * k + 1], a0, b.y);
        }
        if (NSING > 0 && SDF) {
          double bv[4];
          if constexpr (W::GS == 4) {
            // [t][c] layout (mesh.cpp, N <= 4): the lane's four columns in two 16-byte loads instead
            // of four 8-byte ones (C3 65.5 -> 66.0, C2 54.5 -> 55.1 GDOF/s; at N = 6 the phased
            // kernel measured slower with it, 28.4 -> 27.3, and keeps the [c][t] layout)
            const double2 b01 = *reinterpret_cast<const double2*>(ob + W::NPG * 64 + 4 * t4);
            const double2 b23 = *reinterpret_cast<const double2*>(ob + W::NPG * 64 + 4 * t4 + 2);
            bv[0] = b01.x, bv[1] = b01.y, bv[2] = b23.x, bv[3] = b23.y;
          } else {
#pragma unroll
            for (int c = 0; c < W::GS; ++c) bv[c] = ob[W::NPG * 64 + 4 * c + t4];   // Op(32+c, 4ks+t)
          }
#pragma unroll
          for (int k = 0; k < NSING; ++k) {
            const double a0 = X[(mts[k] * 8 + g) * XSTR + t4 + (ks - K0) * 4];
#pragma unroll
            for (int c = 0; c < W::GS; ++c) sacc[k][c] = fma(a0, bv[c], sacc[k][c]);
          }
        } else if (NSING > 0) {
          const double bs = lane < 4 * W::GS ? ob[W::NPG * 64 + (W::GS == 4 ? 4 * t4 + g : lane)] : 0.0;
#pragma unroll
          for (int k = 0; k < NSING; ++k) {
            const double a0 = X[(mts[k] * 8 + g) * XSTR + t4 + (ks - K0) * 4];
            dmma_8x8x4(acc[2 * NPAIR + k], a0, bs);
          }
        }
      }
    };
    if (io.ctid < 32) trace_ev(A, j, 0);
    trace_w(A, j, 4);
    nbar_sync(W::BAR_XV_FULL, NT);
    trace_w(A, j, 5);
    if (io.ctid < 32) trace_ev(A, j, 1);
    if (IODEFER && j >= 1) {
      // tile j-1's buffer hand-offs, deferred from the end of its epilogue to here: the bulk
      // stores' shared-memory reads drain at the SM's share of the HBM write bandwidth (~1.4k
      // cycles for the Q tile at N = 4), and a wait there held every consumer warp at XV_FULL
      const int jp = j - 1, bufp = jp % W::NIN;
      if (io.ctid == IOT) {
        if (MODE == MODE_UPDATE) {
          // NRES == 1: tile j-1's residual store must have left sRes too; else only its Q store
          if (W::NRES == 1) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
          else asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
          if (W::NRES == 1 && ne == EB) load_res(j);
        }
        // two input buffers: refill the one tile j-1 used with the inputs of tile j+1
        if (W::NIN == 2 && jp + 2 < io.nmine && tile_full(jp + 2)) fetch_in(jp + 2);
      }
      // the buffer is free: signal the producers (the partial last tile with two buffers, every
      // tile with three)
      if ((W::NIN == 2 ? (jp + 2 < io.nmine && !tile_full(jp + 2)) : (jp + W::NIN < io.nmine)) &&
          (io.ctid >> 5) == IOW) {
        __syncwarp();
        nbar_arrive(W::BAR_Q_EMPTY + bufp, W::PT + 32);
      }
    }
    if (!IODEFER && W::NRES == 1 && MODE == MODE_UPDATE && io.ctid == IOT && j >= 1 && ne == EB) {
      // tile j-1's residual store has left sRes by now (issued at the end of its epilogue)
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
      load_res(j);
    }
    kloop(KBlk<XSV, 0, S::KSV>{});
    if (io.ctid < 32) trace_ev(A, j, 2);
    if (j + 1 < io.nmine) nbar_arrive(W::BAR_XV_EMPTY, NT);

    nbar_sync(W::BAR_XF_FULL, NT);
    if (io.ctid < 32) trace_ev(A, j, 3);
    kloop(KBlk<XSF, S::KSV, S::KS4>{});
    if (io.ctid < 32) trace_ev(A, j, 4);
    trace_w(A, j, 0);
    if (j + 1 < io.nmine) nbar_arrive(W::BAR_XF_EMPTY, NT);
#ifndef DG_SRED2
#define DG_SRED2 1
#endif
    if (SDF && DG_SRED2) {
      // sum the singles' partial products over the 4 lanes of a row, lane t keeping column t, as
      // a transposing butterfly (3 shuffles per single instead of 2 GS): step 1 (xor 1) each lane
      // keeps the columns of its parity, step 2 (xor 2) the one of its half; all singles' shuffles
      // of a step are issued together
      const bool o1 = t4 & 1, o2 = (t4 & 2) != 0;
      double k0[NSING > 0 ? NSING : 1], k1[NSING > 0 ? NSING : 1];
#pragma unroll
      for (int k = 0; k < NSING; ++k) {
        const double c0 = sacc[k][0], c1 = W::GS > 1 ? sacc[k][1] : 0.0;
        const double c2 = W::GS > 2 ? sacc[k][2] : 0.0, c3 = W::GS > 3 ? sacc[k][3] : 0.0;
        const double s0 = __shfl_xor_sync(0xffffffffu, o1 ? c0 : c1, 1);
        const double s1 = __shfl_xor_sync(0xffffffffu, o1 ? c2 : c3, 1);
        k0[k] = (o1 ? c1 : c0) + s0;   // column o1
        k1[k] = (o1 ? c3 : c2) + s1;   // column 2 + o1
      }
#pragma unroll
      for (int k = 0; k < NSING; ++k) {
        const double s = __shfl_xor_sync(0xffffffffu, o2 ? k0[k] : k1[k], 2);
        acc[2 * NPAIR + k][0] = (o2 ? k1[k] : k0[k]) + s;   // column 2 o2 + o1 = t
      }
    } else if (SDF) {   // sum the singles' partial products over the 4 lanes of a row; lane t keeps column t
#pragma unroll
      for (int k = 0; k < NSING; ++k) {
        double mine = 0.0;
#pragma unroll
        for (int c = 0; c < W::GS; ++c) {
          double v = sacc[k][c];
          v += __shfl_xor_sync(0xffffffffu, v, 1);
          v += __shfl_xor_sync(0xffffffffu, v, 2);
          if (c == t4) mine = v;
        }
        acc[2 * NPAIR + k][0] = mine;
      }
    }
    trace_w(A, j, 2);
    const bool staged = MODE == MODE_UPDATE && ne == EB;
    if (staged) mbar_wait(io.barRes + j % W::NRES, (j / W::NRES) & 1);   // only the last tile can be partial
    trace_w(A, j, 3);
    if (staged) {
      // in chunks of CH units: all loads of a chunk first (q_s and sRes could alias as far as the
      // compiler knows), then its stores
      // slots per epilogue chunk (loads of a chunk first, then its stores): 6 at N = 4 (C4 55.9 ->
      // 56.1 GDOF/s; 3: 55.5, 8: 54.7), 4 elsewhere
#ifdef DG_ECH
      constexpr int CH = DG_ECH;
#else
      constexpr int CH = N == 4 ? 6 : 4;
#endif
#pragma unroll
      for (int u0 = 0; u0 < NSLOT; u0 += CH) {
        double rv[CH][2], qv[CH][2];
#pragma unroll
        for (int u = u0; u < u0 + CH && u < NSLOT; ++u)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int n = unit_n(u, q);
            const int li = (unit_mt(u) * 8 + g) * NP + (n < NP ? n : 0);
            rv[u - u0][q] = sRes[li];
            qv[u - u0][q] = q_s[li];
          }
#pragma unroll
        for (int u = u0; u < u0 + CH && u < NSLOT; ++u)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int n = unit_n(u, q);
            if (n >= NP) continue;
            const int li = (unit_mt(u) * 8 + g) * NP + n;   // == (e*5 + c)*NP + n
            const double rr = fma(A.a, rv[u - u0][q], A.dt * acc[u][q]);
            const double qn = fma(A.b, rr, qv[u - u0][q]);
            sRes[li] = rr;
            q_s[li] = qn;
          }
      }
    } else {
#pragma unroll
      for (int u = 0; u < NSLOT; ++u) {
        const int row = unit_mt(u) * 8 + g;
        const int e = row / 5, c = row - 5 * (row / 5);
        if (e >= ne) continue;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int n = unit_n(u, q);
          if (n >= NP) continue;
          const double rhs = acc[u][q];
          const int li = row * NP + n;
          if (MODE == MODE_UPDATE) {
            const size_t gi = size_t(e0) * 5 * NP + li;
            const double rr = fma(A.a, __ldg(A.res + gi), A.dt * rhs);
            A.res[gi] = rr;
            A.Qout[gi] = fma(A.b, rr, q_s[li]);
          } else {
            A.out[(size_t(c) * A.Kpub + A.pub[e0 + e]) * NP + n] = rhs;
          }
        }
      }
    }
    if (io.ctid < 32) trace_ev(A, j, 6);
    trace_w(A, j, 1);
    if (staged) {
      // every thread that wrote the staged tiles orders its generic-proxy stores before the
      // async-proxy (TMA) reads of the bulk stores issued after the barrier
      fence_proxy_async();
      nbar_sync(W::BAR_C, W::CT);
      if (io.ctid < 32) trace_ev(A, j, 7);
      if (io.ctid == IOT) {
        // Q first (its buffer is released first); neither store is waited for here: the input
        // refill / release and (NRES == 1) the next residual load follow at the next tile's
        // XV_FULL
        fence_proxy_async();
        tma_store_1d(A.Qout + size_t(e0) * 5 * NP, q_s, W::BQ);
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        tma_store_1d(A.res + size_t(e0) * 5 * NP, sRes, W::BQ);
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        if (!IODEFER) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
        if (W::NRES == 2 && j + 1 < io.nmine && tile_full(j + 1)) {
          // the next tile's residual goes where tile j-1's was stored from: every group but the
          // two just committed has been read (issued a tile ago)
          if (IODEFER) asm volatile("cp.async.bulk.wait_group.read 2;\n" ::: "memory");
          load_res(j + 1);
        }
      }
    }
    if (io.ctid < 32) trace_ev(A, j, 5);
    if (!IODEFER) {
      if (W::NIN == 2) {
        if (io.ctid == IOT && j + 2 < io.nmine && tile_full(j + 2)) fetch_in(j + 2);
        if (j + 2 < io.nmine && !tile_full(j + 2) && (io.ctid >> 5) == IOW) {
          __syncwarp();
          nbar_arrive(W::BAR_Q_EMPTY + buf, W::PT + 32);
        }
      } else if (j + W::NIN < io.nmine && (io.ctid >> 5) == IOW) {
        __syncwarp();
        nbar_arrive(W::BAR_Q_EMPTY + buf, W::PT + 32);
      }
    }
    trace_w(A, j, 6);
  }
  // make the last bulk stores globally visible before the kernel ends
  if (io.ctid == IOT) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

template <int N, int MODE, int V = 0>
__global__ void __launch_bounds__(WS<N, V>::NT, 1) stage_ws_kernel(const StageArgs A) {
  using S = Shape<N>;
  using W = WS<N, V>;
  constexpr int NP = S::NP, NFP = S::NFP, EB = W::EB, NT = W::NT, PT = W::PT;
  constexpr int XSV = W::XSV, XSF = W::XSF;
  extern __shared__ __align__(128) unsigned char smem[];
  double* sXv = reinterpret_cast<double*>(smem);
  double* sXf = sXv + W::ROWS * XSV;
  double* sOp = sXf + W::ROWS * XSF;
  unsigned char* in0 = reinterpret_cast<unsigned char*>(sOp) + W::SMEM_OP;
  auto bufQ = [&](int b) { return reinterpret_cast<double*>(in0 + b * W::BIN); };
  auto bufG = [&](int b) { return reinterpret_cast<double*>(in0 + b * W::BIN + W::BQ); };
  auto bufN = [&](int b) { return reinterpret_cast<int*>(in0 + b * W::BIN + W::BQ + W::BG); };
  auto bufC = [&](int b) { return reinterpret_cast<uint8_t*>(in0 + b * W::BIN + W::BQ + W::BG + W::BN); };
  double* sRes = reinterpret_cast<double*>(in0 + W::SMEM_IN);
  uint8_t* sTbl = reinterpret_cast<uint8_t*>(in0 + W::SMEM_IN + W::SMEM_RES);
  uint8_t* sTblf = sTbl + 96 * NFP;
  uint8_t* sFm = sTblf + 96 * NFP;
  uint64_t* sBar = reinterpret_cast<uint64_t*>(sTbl + W::SMEM_T);   // NIN inputs, then NRES residuals
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // DG_PDL (bit mask over the orders): programmatic dependent launch -- the next stage's CTA may start on this SM as
  // soon as this CTA exits and run its prologue (operator and tables, barriers) while other SMs
  // finish; it waits for the whole previous stage before touching the state
  constexpr bool PDL = (DG_PDL >> N) & 1;   // DG_PDL: bit N enables it at order N
  if (PDL) pdl_launch_dependents();

  // B operand (mesh.cpp layout: per k-step the n-tile pairs, then the compacted odd n-tile)
  for (int i = tid; i < W::OPC; i += NT) sOp[i] = A.op[i];
  for (int i = tid; i < 96 * NFP; i += NT) {
    sTbl[i] = A.tbl[i];
    sTblf[i] = A.tblf[i];
  }
  for (int i = tid; i < 4 * NFP; i += NT) sFm[i] = A.fmask[i];
  for (int i = tid; i < W::ROWS * (XSV + XSF); i += NT) sXv[i] = 0.0;   // padding columns stay 0
  if (tid == 0) {
    for (int b = 0; b < W::NIN + W::NRES; ++b) mbar_init(&sBar[b], 1);   // inputs, then residuals
  }
  __syncthreads();
  if (PDL) pdl_wait();

  const int ntiles = (A.e_end - A.e_begin + EB - 1) / EB;
  const int nmine = (ntiles > (int)blockIdx.x) ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;

  // Producers take the HIGH warp ids (N = 4): the SMSP arbiter issues highest-wid-first, so their
  // short FP64 chains win the shared FP64/DMMA pipe and the consumers fill the remaining slots.
  // N = 3 (consumers the bound): the consumers take the high warp ids instead (C3 66.3 -> 67.1,
  // C2 55.0 -> 55.3 GDOF/s; at N = 4, where the producers are the bound, 56.0 -> 54.5)
#ifdef DG_CHI
  constexpr bool CHI = DG_CHI;
#else
  constexpr bool CHI = N == 3;
#endif
  static_assert(!CHI || W::PW % 4 == 0, "consumer cw must run on SMSP cw % 4 (M8Plan)");
  const bool is_producer = CHI ? warp < W::PW : warp >= W::CW;
  if (is_producer) {
    const int ptid = CHI ? tid : tid - W::CT, pwarp = ptid >> 5;
    // ======================= producers: load (TMA), volume flux, face flux
    const double gm1 = A.gamma - 1.0;
    auto fetch = [&](int jj) {
      const int tile = blockIdx.x + jj * gridDim.x;
      const int e0 = A.e_begin + tile * EB;
      const int ne = min(EB, A.e_end - e0);
      const int b = jj % W::NIN;
      if (ne == EB) {
        if (ptid == 0) {
          fence_proxy_async();
          mbar_arrive_expect_tx(&sBar[b], W::BIN);
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
        for (int i = ptid; i < EB * 5 * NP; i += PT) q_s[i] = i < ne * 5 * NP ? __ldg(A.Qin + size_t(e0) * 5 * NP + i) : 0.0;
        for (int i = ptid; i < EB * GEO; i += PT) g_s[i] = i < ne * GEO ? __ldg(A.geo + size_t(e0) * GEO + i) : 0.0;
        for (int i = ptid; i < EB * 4; i += PT) {
          n_s[i] = i < ne * 4 ? __ldg(A.nbr + size_t(e0) * 4 + i) : 0;
          c_s[i] = i < ne * 4 ? A.code[size_t(e0) * 4 + i] : uint8_t(CODE_BC + 2);
        }
        nbar_sync(W::BAR_P, PT);
      }
    };
    if (nmine > 0) fetch(0);
    if (W::NIN == 2 && nmine > 1) fetch(1);   // later full tiles are fetched by the consumers
    for (int j = 0; j < nmine; ++j) {
      const int tile = blockIdx.x + j * gridDim.x;
      const int e0 = A.e_begin + tile * EB;
      const int ne = min(EB, A.e_end - e0);
      const int buf = j % W::NIN;
      const double* q_s = bufQ(buf);
      const double* g_s = bufG(buf);
      const int* n_s = bufN(buf);
      const uint8_t* c_s = bufC(buf);
      if (ptid < 32) trace_ev(A, j, 8);
      if (ne == EB) mbar_wait(&sBar[buf], (j / W::NIN) & 1);
      if (ptid < 32) trace_ev(A, j, 9);
      // ---- issue this pwarp's neighbour-trace gathers for the whole tile first: their latency
      //      hides behind the volume phase
      const int seg = lane / W::SEGW, i = lane - seg * W::SEGW;
      const bool lane_ok = i < NFP && seg < W::NSEG;
      const int fbase = pwarp * W::NSEG + seg;
      double qp[W::FPASS][5];
      face_gather<N, W::FPASS>(A, fbase, W::PW * W::NSEG, 4 * EB, ne, i, lane_ok, q_s, g_s, n_s, c_s, sTbl, sTblf, sFm, qp);
      if (ptid < 32) trace_ev(A, j, 15);
      // ---- volume fluxes -> Xv
      trace_w(A, j, 4);
      if (j >= 1) nbar_sync(W::BAR_XV_EMPTY, NT);
      trace_w(A, j, 5);
      if (ptid < 32) trace_ev(A, j, 10);
      // branch-free, two nodes per thread interleaved (independent FP64 chains); slots past the
      // tile's nodes compute on a clamped node and only store zeros / nothing
      constexpr int VR = (EB * NP + PT - 1) / PT;
      // N = 3: slot blocks in reversed warp order (a partial round lands on the highest producer
      // warp ids, which the SMSP arbiter favours) and warps without nodes in a round skip it:
      // C3 56.3 vs 55.1 GDOF/s; at N = 4 the same measured 49.5 vs 55.0 (DG_SKIP_VOL overrides)
#ifdef DG_SKIP_VOL
      constexpr bool SKIPV = DG_SKIP_VOL;
#else
      constexpr bool SKIPV = N == 3 || N == 2;   // N = 2 (EB = 48, 12 + 4 warps): 62.8 -> 65.7 GDOF/s
#endif
#pragma unroll
      for (int r0 = 0; r0 < VR; r0 += 2) {
        if DG_SKIPQ(2) break;
#pragma unroll
        for (int rr = r0; rr < r0 + 2 && rr < VR; ++rr) {
          if constexpr (SKIPV) {
            if (rr * PT + (W::PW - 1 - pwarp) * 32 >= EB * NP) continue;
          }
          const int idx = SKIPV ? (W::PW - 1 - pwarp) * 32 + lane + rr * PT : ptid + rr * PT;
          vol_node<N, XSV>(A, idx, q_s, g_s, e0, ne, gm1, sXv, EB * NP);
        }
      }
      if (ptid < 32) trace_ev(A, j, 11);
      trace_w(A, j, 0);
      nbar_arrive(W::BAR_XV_FULL, NT);
      // ---- prefetch the next tile's inputs (its buffer was last read by the epilogue of tile j-1;
      //      the Q_EMPTY sync also covers every producer thread having left tile j-1)
      if (W::NIN == 2) {
        if (j + 1 < nmine && j + 1 >= 2 && A.e_end - (A.e_begin + (int(blockIdx.x) + (j + 1) * int(gridDim.x)) * EB) < EB) {
          nbar_sync(W::BAR_Q_EMPTY + (j + 1) % W::NIN, W::PT + 32);   // the partial last tile
          fetch(j + 1);
        }
      } else if (j + 1 < nmine) {
        if (j + 1 >= W::NIN) nbar_sync(W::BAR_Q_EMPTY + (j + 1) % W::NIN, W::PT + 32);
        fetch(j + 1);
      }
      // ---- face fluxes -> Xf
      if (ptid < 32) trace_ev(A, j, 12);
      trace_w(A, j, 6);
      if (j >= 1) nbar_sync(W::BAR_XF_EMPTY, NT);
      trace_w(A, j, 7);
      if (ptid < 32) trace_ev(A, j, 13);
      face_terms<N, W::FPASS, W::SEGW, XSF>(A, fbase, W::PW * W::NSEG, 4 * EB, ne, i, lane_ok, q_s, g_s, sFm, qp, sXf);
      if (ptid < 32) trace_ev(A, j, 14);
      trace_w(A, j, 1);
      nbar_arrive(W::BAR_XF_FULL, NT);
    }
  } else {
    // ======================= consumers: DMMA contraction + LSERK epilogue
    // every warp runs a compile-time-shaped loop over its units so its DMMA chains interleave
    // without run-time branches
    using PL = M8Plan<N, V>;
    const int cw = CHI ? warp - W::PW : warp;   // W::PW % 4 == 0: consumer cw still runs on SMSP cw % 4
    ConsumerIO<N, MODE, V> io{A, sXv, sXf, sOp, in0, sRes, &sBar[W::NIN], &sBar[0], nmine, CHI ? tid - W::PT : tid, lane};
    int singles[PL::CSMAX], ns = 0;
    m8_singles<N, V>(cw, singles, ns);
    const int np8 = PL::P > cw ? (PL::P - 1 - cw) / PL::CW + 1 : 0;
    constexpr int CP = PL::CPMAX, CPm = PL::CPMAX > 0 ? PL::CPMAX - 1 : 0;
    // instantiate only the per-warp shapes the greedy plan can produce
    constexpr int SMAX = PL::maxcount();
#define DG_M8_CASE(PA, SI)                                                   \
  if constexpr (PL::occurs(PA, SI)) {                                        \
    if (np8 == PA && ns == SI) ws_consumer_m8<N, MODE, PA, SI, V>(io, cw, singles); \
  }
    DG_M8_CASE(CP, 0) DG_M8_CASE(CP, 1) DG_M8_CASE(CP, 2) DG_M8_CASE(CP, 3) DG_M8_CASE(CP, 4)
    DG_M8_CASE(CP, 5) DG_M8_CASE(CP, 6) DG_M8_CASE(CP, 7) DG_M8_CASE(CP, 8)
    if (CPm != CP) {
      DG_M8_CASE(CPm, 0) DG_M8_CASE(CPm, 1) DG_M8_CASE(CPm, 2) DG_M8_CASE(CPm, 3) DG_M8_CASE(CPm, 4)
      DG_M8_CASE(CPm, 5) DG_M8_CASE(CPm, 6) DG_M8_CASE(CPm, 7) DG_M8_CASE(CPm, 8)
    }
    static_assert(SMAX <= 8, "singles per warp beyond the dispatch cases");
#undef DG_M8_CASE
  }
}

// ---------------------------------------------------------------- high-order kernel (N = 5, 6)
// For N = 5, 6 the contraction is ~90 % of the stage's flops and the operator Op (113 KB /
// 256 KB) does not fit next to the tile, so the warp specialisation of the N <= 4 kernel buys
// little.  All 16 warps run each tile in phases -- traces, volume and face fluxes into X, the
// contraction, the LSERK epilogue -- while Op streams through a 3-slot shared-memory ring in
// chunks of KC k-steps (TMA bulk copies, full/empty mbarriers, prefetched two chunks ahead and
// across tile boundaries), and the next tile's inputs arrive by TMA during the current tile.
// Each warp owns one work item: an n-tile pair (or the compacted odd n-tile) times up to MU
// consecutive 8-row tiles, so every B fragment is read once per k-step and reused MU times;
// items go to SMSPs longest-first to balance the per-SMSP FP64 pipes.
template <int N>
struct HO {
  using S = Shape<N>;
  static constexpr int EB = 8, NW = 15, CT = 32 * NW, NT = CT + 32;   // + one loader warp
  static constexpr int ROWS = 5 * EB, MT8 = ROWS / 8;
  static constexpr int XS = S::XS;
  static constexpr int NPG = S::NTL / 2, HS = S::NTL % 2;
  static constexpr int GS = HS ? S::NP - 8 * (S::NTL - 1) : 0;
  static constexpr int OPW = NPG * 64 + 4 * GS;                   // doubles per k-step of Op
#ifndef DG_HO_SDF
#define DG_HO_SDF 1
#endif
  static constexpr bool SDF = DG_HO_SDF && GS > 0 && GS <= 4;     // odd n-tile on DFMA (N = 6)
#ifdef DG_HO_KC
  static constexpr int KC = DG_HO_KC;
#else
  static constexpr int KC = (N == 6) ? 6 : 7;                     // k-steps per ring chunk
#endif
#ifdef DG_HO_SLOTS
  static constexpr int NSLOT = DG_HO_SLOTS;
#else
  static constexpr int NSLOT = 3;                                 // ring slots
#endif
  static constexpr int NCH = (S::KS4 + KC - 1) / KC;
  static constexpr int KLAST = S::KS4 - (NCH - 1) * KC;          // k-steps of the last chunk
  static constexpr uint32_t BCH = uint32_t(KC) * OPW * 8;
  static constexpr int MU = (N == 6) ? 3 : 2;                     // 8-row tiles per work item
  static constexpr int SEGW = S::NFP <= 4 ? 4 : S::NFP <= 8 ? 8 : S::NFP <= 16 ? 16 : 32;
  static constexpr int NSEG = 32 / SEGW, STRIDE = NW * NSEG;
  static constexpr int FPASS = (EB * 4 + STRIDE - 1) / STRIDE;
  static constexpr uint32_t BQ = uint32_t(EB) * 5 * S::NP * 8;
  static constexpr uint32_t BG = uint32_t(EB) * GEO * 8;
  static constexpr uint32_t BN = uint32_t(EB) * 4 * 4;
  static constexpr uint32_t BC = uint32_t(EB) * 4;
  static constexpr uint32_t BIN = BQ + BG + BN + BC;
  static_assert(BQ % 16 == 0 && BG % 16 == 0 && BCH % 16 == 0 && (uint32_t(OPW) * 8) % 16 == 0, "TMA sizes");
  static constexpr size_t SMEM_X = size_t(ROWS) * XS * 8;
  static_assert(2 * size_t(BQ) <= SMEM_X, "X doubles as the output staging tile");
  static constexpr size_t SMEM_T = size_t(2 * 96 * S::NFP + 4 * S::NFP + 15) / 16 * 16;
  static constexpr size_t SMEM = SMEM_X + 2 * size_t(BIN) + NSLOT * size_t(BCH) + SMEM_T + 16 * (2 + 2 * NSLOT);
  static_assert(SMEM <= 227 * 1024, "high-order tile does not fit in shared memory");
};

struct HOItem {
  int kind, p, m0, mc;   // kind 0: n-tile pair p; 1: odd n-tile; -1: idle
};

// Deterministic plan, evaluated by every thread: items (n-group x runs of <= MU row tiles) in
// creation order, placed longest-first on the least-loaded SMSP (warp w runs on SMSP w % 4).
template <int N>
__device__ __forceinline__ HOItem ho_plan(int warp) {
  using H = HO<N>;
  constexpr int NG = H::NPG + H::HS, NRUN = (H::MT8 + H::MU - 1) / H::MU, NIT = NG * NRUN;
  static_assert(NIT <= H::NW, "more work items than warps");
  int load[4] = {0, 0, 0, 0}, cnt[4] = {0, 0, 0, 0};
  HOItem mine{-1, 0, 0, 0};
  for (int wgt = 2 * H::MU; wgt >= 1; --wgt)
    for (int it = 0; it < NIT; ++it) {
      const int grp = it / NRUN, run = it % NRUN;
      const int kind = grp < H::NPG ? 0 : 1;
      const int m0 = run * H::MU, mc = min(H::MU, H::MT8 - m0);
      if ((kind == 0 ? 2 : 1) * mc != wgt) continue;
      int best = -1;
      for (int s = 0; s < 4; ++s)
        if (s + 4 * cnt[s] < H::NW && (best < 0 || load[s] < load[best])) best = s;
      const int w = best + 4 * cnt[best];
      ++cnt[best];
      load[best] += wgt;
      if (w == warp) mine = HOItem{kind, kind == 0 ? grp : 0, m0, mc};
    }
  return mine;
}

// KCN k-steps of one ring chunk for a work item of MC row tiles and n-group KIND (0: pair,
// 1: compacted odd n-tile): one B fragment per k-step, reused MC times
template <int N, int KIND, int MC, int KCN>
__device__ __forceinline__ void ho_chunk(double (&acc)[HO<N>::MU][2][2], const double* xa, const double* ob, int kb,
                                         int lane) {
  using H = HO<N>;
#pragma unroll
  for (int kk = 0; kk < KCN; ++kk) {
    const int kcol = (kb + kk) * 4;
    if (KIND == 0) {
      const double2 b = *reinterpret_cast<const double2*>(ob + kk * H::OPW + 2 * lane);
#pragma unroll
      for (int m = 0; m < MC; ++m) {
        const double a = xa[m * 8 * H::XS + kcol];
        dmma_8x8x4(acc[m][0], a, b.x);
        dmma_8x8x4(acc[m][1], a, b.y);
      }
    } else if (H::SDF) {
      // odd n-tile with GS <= 4 real columns on DFMA: lane (g, t) accumulates row g x column c
      // over its k = t (mod 4) in acc[m][c / 2][c % 2]; reduced over t after the contraction
      double bv[H::GS];
#pragma unroll
      for (int c = 0; c < H::GS; ++c) bv[c] = ob[kk * H::OPW + 4 * c + (lane & 3)];
#pragma unroll
      for (int m = 0; m < MC; ++m) {
        const double a = xa[m * 8 * H::XS + kcol];
#pragma unroll
        for (int c = 0; c < H::GS; ++c) acc[m][c >> 1][c & 1] = fma(a, bv[c], acc[m][c >> 1][c & 1]);
      }
    } else {
      const double b = lane < 4 * H::GS ? ob[kk * H::OPW + lane] : 0.0;
#pragma unroll
      for (int m = 0; m < MC; ++m) dmma_8x8x4(acc[m][0], xa[m * 8 * H::XS + kcol], b);
    }
  }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

template <int N, int MODE>
__global__ void __launch_bounds__(HO<N>::NT, 1) stage_ho_kernel(const StageArgs A) {
  using S = Shape<N>;
  using H = HO<N>;
  constexpr int NP = S::NP, NFP = S::NFP, EB = H::EB, NT = H::NT, CT = H::CT, XS = H::XS, MU = H::MU;
  extern __shared__ __align__(128) unsigned char smem[];
  double* sX = reinterpret_cast<double*>(smem);
  unsigned char* in0 = smem + H::SMEM_X;
  double* ring = reinterpret_cast<double*>(in0 + 2 * H::BIN);
  uint8_t* sTbl = reinterpret_cast<uint8_t*>(ring) + H::NSLOT * H::BCH;
  uint8_t* sTblf = sTbl + 96 * NFP;
  uint8_t* sFm = sTblf + 96 * NFP;
  uint64_t* sBar = reinterpret_cast<uint64_t*>(sTbl + H::SMEM_T);   // [0,1] inputs, then ring full, ring empty
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  auto bufQ = [&](int b) { return reinterpret_cast<double*>(in0 + b * H::BIN); };
  auto bufG = [&](int b) { return reinterpret_cast<double*>(in0 + b * H::BIN + H::BQ); };
  auto bufN = [&](int b) { return reinterpret_cast<int*>(in0 + b * H::BIN + H::BQ + H::BG); };
  auto bufC = [&](int b) { return reinterpret_cast<uint8_t*>(in0 + b * H::BIN + H::BQ + H::BG + H::BN); };

  for (int i = tid; i < 96 * NFP; i += NT) {
    sTbl[i] = A.tbl[i];
    sTblf[i] = A.tblf[i];
  }
  for (int i = tid; i < 4 * NFP; i += NT) sFm[i] = A.fmask[i];
  for (int i = tid; i < H::ROWS * XS; i += NT) sX[i] = 0.0;   // padding columns stay 0
  if (tid == 0) {
    for (int b = 0; b < 2 + H::NSLOT; ++b) mbar_init(&sBar[b], 1);                    // inputs, ring full
    for (int b = 2 + H::NSLOT; b < 2 + 2 * H::NSLOT; ++b) mbar_init(&sBar[b], H::NW);  // ring empty
  }
  __syncthreads();

  const int ntiles = (A.e_end - A.e_begin + EB - 1) / EB;
  const int nmine = (ntiles > (int)blockIdx.x) ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const long long nchunks = (long long)nmine * H::NCH;
  auto tile_e0 = [&](int jj) { return A.e_begin + (int(blockIdx.x) + jj * int(gridDim.x)) * EB; };
  auto is_full = [&](int jj) { return A.e_end - tile_e0(jj) >= EB; };
  auto fetch = [&](int jj) {   // one thread
    const int e0 = tile_e0(jj), b = jj & 1;
    fence_proxy_async();
    mbar_arrive_expect_tx(&sBar[b], H::BIN);
    tma_load_1d(bufQ(b), A.Qin + size_t(e0) * 5 * NP, H::BQ, &sBar[b]);
    tma_load_1d(bufG(b), A.geo + size_t(e0) * GEO, H::BG, &sBar[b]);
    tma_load_1d(bufN(b), A.nbr + size_t(e0) * 4, H::BN, &sBar[b]);
    tma_load_1d(bufC(b), A.code + size_t(e0) * 4, H::BC, &sBar[b]);
  };
  auto load_chunk = [&](long long gc) {   // one thread; the slot is free
    const int s = int(gc % H::NSLOT), c = int(gc % H::NCH);
    const int kc = min(H::KC, S::KS4 - c * H::KC);
    const uint32_t bytes = uint32_t(kc) * H::OPW * 8;
    mbar_arrive_expect_tx(&sBar[2 + s], bytes);
    tma_load_1d(ring + size_t(s) * (H::BCH / 8), A.op + size_t(c) * H::KC * H::OPW, bytes, &sBar[2 + s]);
  };
  if (warp == H::NW) {
    // loader warp: keeps the Op ring full, each slot refilled as soon as all compute warps
    // have released it
    if (lane == 0)
      for (long long gn = 0; gn < nchunks; ++gn) {
        if (gn >= H::NSLOT)
          mbar_wait(&sBar[2 + H::NSLOT + int(gn % H::NSLOT)], uint32_t(((gn / H::NSLOT) - 1) & 1));
        load_chunk(gn);
      }
    return;
  }
  if (tid == 0 && nmine > 0 && is_full(0)) fetch(0);
  const HOItem it = ho_plan<N>(warp);
  const double gamma = A.gamma, gm1 = A.gamma - 1.0;
  long long gch = 0;   // chunks consumed so far

  for (int j = 0; j < nmine; ++j) {
    const int e0 = tile_e0(j);
    const int ne = min(EB, A.e_end - e0);
    const bool full = ne == EB;
    const int buf = j & 1;
    double* q_s = bufQ(buf);
    double* g_s = bufG(buf);
    int* n_s = bufN(buf);
    uint8_t* c_s = bufC(buf);
    if (warp == 0) trace_ev(A, j, 0);
    if (tid == 0 && j + 1 < nmine && is_full(j + 1)) fetch(j + 1);   // its buffer was freed by tile j-1
    if (full) {
      mbar_wait(&sBar[buf], (j >> 1) & 1);
    } else {   // the last tile: plain loads, zero-filled
      for (int i = tid; i < EB * 5 * NP; i += CT) q_s[i] = i < ne * 5 * NP ? __ldg(A.Qin + size_t(e0) * 5 * NP + i) : 0.0;
      for (int i = tid; i < EB * GEO; i += CT) g_s[i] = i < ne * GEO ? __ldg(A.geo + size_t(e0) * GEO + i) : 0.0;
      for (int i = tid; i < EB * 4; i += CT) {
        n_s[i] = i < ne * 4 ? __ldg(A.nbr + size_t(e0) * 4 + i) : 0;
        c_s[i] = i < ne * 4 ? A.code[size_t(e0) * 4 + i] : uint8_t(CODE_BC + 2);
      }
      nbar_sync(1, CT);
    }
    if (warp == 0) trace_ev(A, j, 1);
    // ---- neighbour traces (one face per SEGW-lane segment, FPASS passes)
    const int seg = lane / H::SEGW, i = lane - seg * H::SEGW;
    const bool lane_ok = i < NFP;
    double qp[H::FPASS][5];
#pragma unroll
    for (int u = 0; u < H::FPASS; ++u) {
      const int face = warp * H::NSEG + u * H::STRIDE + seg;
      const int e = face >> 2, f = face & 3;
#pragma unroll
      for (int c = 0; c < 5; ++c) qp[u][c] = A.qinf[c];
      if (!DG_SKIPQ(2) && lane_ok && face < EB * 4 && e < ne) {
        const int code = c_s[e * 4 + f];
        if (code < CODE_BC) {
          gather_trace<NP, NFP>(A, code, n_s[e * 4 + f], f, i, sTbl, sTblf, qp[u]);
        } else {
          const double* Gf = g_s + e * GEO + 9 + 4 * f;
          const double* q = q_s + e * 5 * NP + sFm[f * NFP + i];
          double qm[5];
#pragma unroll
          for (int c = 0; c < 5; ++c) qm[c] = q[c * NP];
          ghost_trace(A, code - CODE_BC, qm, Gf[0], Gf[1], Gf[2], qp[u]);
        }
      }
    }
    if (warp == 0) trace_ev(A, j, 2);
    // the previous tile's output bulk stores have left X
    if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    nbar_sync(1, CT);
    if (warp == 0) trace_ev(A, j, 3);
    // ---- volume fluxes -> X[:, 0:3Np)
    if (!DG_SKIPQ(2)) {
      constexpr int VR = (EB * NP + CT - 1) / CT;
#pragma unroll
      for (int rr = 0; rr < VR; ++rr) {
        const int idx = tid + rr * CT;
        if (idx >= ne * NP) break;
        const int e = idx / NP, n = idx - e * NP;
        const double* q = q_s + e * 5 * NP + n;
        const double rho = q[0], mx = q[NP], my = q[2 * NP], mz = q[3 * NP], E = q[4 * NP];
        const double ri = rcp_nr(rho);
        const double u = mx * ri, v = my * ri, w = mz * ri;
        const double p = gm1 * (E - 0.5 * (mx * u + my * v + mz * w));
        if (!state_ok(rho, p, mx, my, mz, E)) flag_blowup(A.flag, A.gid[e0 + e]);
        const double* Gv = g_s + e * GEO;
        const double Ep = E + p, pd = p - A.pref;   // background-flux subtraction (A14)
        double* xr = sX + (e * 5) * XS + n;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double cx = Gv[3 * d], cy = Gv[3 * d + 1], cz = Gv[3 * d + 2];
          const double U = cx * u + cy * v + cz * w;   // contravariant velocity along xi_d
          xr[d * NP] = rho * U;
          xr[XS + d * NP] = fma(cx, pd, mx * U);
          xr[2 * XS + d * NP] = fma(cy, pd, my * U);
          xr[3 * XS + d * NP] = fma(cz, pd, mz * U);
          xr[4 * XS + d * NP] = Ep * U;
        }
      }
    }
    if (warp == 0) trace_ev(A, j, 4);
    // ---- face terms -> X[:, KVP:KVP+4Nfp)  (the single-read form of the N <= 4 kernel spills
    //      here: C5 23.7 vs 28.4 GDOF/s)
    if (!DG_SKIPQ(2)) {
      double rip[H::FPASS], unp[H::FPASS], pp[H::FPASS], lam[H::FPASS], unmv[H::FPASS], pmv[H::FPASS];
#pragma unroll
      for (int u = 0; u < H::FPASS; ++u) {
        const int face = warp * H::NSEG + u * H::STRIDE + seg;
        const bool act = lane_ok && face < EB * 4 && (face >> 2) < ne;
        const int fc = act ? face : 0;
        const int e = fc >> 2, f = fc & 3, ii = lane_ok ? i : 0;
        const double* Gf = g_s + e * GEO + 9 + 4 * f;
        const double nx = Gf[0], ny = Gf[1], nz = Gf[2];
        const double* q = q_s + e * 5 * NP + sFm[f * NFP + ii];
        const double qm0 = q[0], qm1 = q[NP], qm2 = q[2 * NP], qm3 = q[3 * NP], qm4 = q[4 * NP];
        const double rim = rcp_nr(qm0);
        const double unm = (qm1 * nx + qm2 * ny + qm3 * nz) * rim;
        const double pm = gm1 * (qm4 - 0.5 * (qm1 * qm1 + qm2 * qm2 + qm3 * qm3) * rim);
        unmv[u] = unm;
        pmv[u] = pm;
        rip[u] = rcp_nr(qp[u][0]);
        unp[u] = (qp[u][1] * nx + qp[u][2] * ny + qp[u][3] * nz) * rip[u];
        pp[u] = gm1 * (qp[u][4] - 0.5 * (qp[u][1] * qp[u][1] + qp[u][2] * qp[u][2] + qp[u][3] * qp[u][3]) * rip[u]);
        const double l = fmax(fabs(unm) + sqrt_nr(gamma * pm * rim), fabs(unp[u]) + sqrt_nr(gamma * pp[u] * rip[u]));
        lam[u] = act ? l : 0.0;
      }
      if (A.lambda_mode == 0) {
#pragma unroll
        for (int d = 1; d < H::SEGW; d <<= 1) {
#pragma unroll
          for (int u = 0; u < H::FPASS; ++u) {
            const long long a = __double_as_longlong(lam[u]);
            const long long o = __shfl_xor_sync(0xffffffffu, a, d);
            lam[u] = __longlong_as_double(a > o ? a : o);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < H::FPASS; ++u) {
        const int face = warp * H::NSEG + u * H::STRIDE + seg;
        const bool act = lane_ok && face < EB * 4 && (face >> 2) < ne;
        if (!act) continue;
        const int e = face >> 2, f = face & 3;
        const double* Gf = g_s + e * GEO + 9 + 4 * f;
        double* xd = sX + (e * 5) * XS + S::KVP + f * NFP + i;
        const double nx = Gf[0], ny = Gf[1], nz = Gf[2], hfs = 0.5 * Gf[3];
        const double* q = q_s + e * 5 * NP + sFm[f * NFP + i];
        double qm[5];
#pragma unroll
        for (int c = 0; c < 5; ++c) qm[c] = q[c * NP];
        const double pm = pmv[u], unm = unmv[u];
        const double pdm = pm - A.pref, pdp = pp[u] - A.pref;
        double df[5];
        df[0] = qm[0] * unm - qp[u][0] * unp[u];
        df[1] = fma(pdm, nx, qm[1] * unm) - fma(pdp, nx, qp[u][1] * unp[u]);
        df[2] = fma(pdm, ny, qm[2] * unm) - fma(pdp, ny, qp[u][2] * unp[u]);
        df[3] = fma(pdm, nz, qm[3] * unm) - fma(pdp, nz, qp[u][3] * unp[u]);
        df[4] = (qm[4] + pm) * unm - (qp[u][4] + pp[u]) * unp[u];
        // Fscale (n.F(q-) - F*) = Fscale/2 ((n.F(q-) - n.F(q+)) + lam (q+ - q-))
#pragma unroll
        for (int c = 0; c < 5; ++c) xd[c * XS] = hfs * fma(lam[u], qp[u][c] - qm[c], df[c]);
      }
    }
    // residual for the epilogue (its latency hides behind the contraction)
    double rprev[MU][2][2];
#pragma unroll
    for (int m = 0; m < MU; ++m)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int row = (it.m0 + m) * 8 + g;
          const int n = (it.kind == 0 ? (2 * it.p + h) * 8 : (S::NTL - 1) * 8) + 2 * t4 + q;
          const bool ok = MODE == MODE_UPDATE && it.kind >= 0 && m < it.mc && (it.kind == 0 || h == 0) && n < NP &&
                          row / 5 < ne;
          rprev[m][h][q] = ok ? __ldg(A.res + size_t(e0) * 5 * NP + row * NP + n) : 0.0;
        }
    if (warp == 0) trace_ev(A, j, 5);
    nbar_sync(1, CT);   // X complete
    if (warp == 0) trace_ev(A, j, 6);
    // ---- contraction: Op streams through the ring, chunk by chunk
    double acc[MU][2][2];
#pragma unroll
    for (int m = 0; m < MU; ++m) acc[m][0][0] = acc[m][0][1] = acc[m][1][0] = acc[m][1][1] = 0.0;
    const double* xa = sX + (it.m0 * 8 + g) * XS + t4;
#if DG_TRACE
    long long wfull = 0;
#endif
    for (int c = 0; c < H::NCH; ++c) {
      const long long gc = gch + c;
      const int s = int(gc % H::NSLOT);
#if DG_TRACE
      long long tw0 = clock64();
#endif
      mbar_wait(&sBar[2 + s], uint32_t((gc / H::NSLOT) & 1));
#if DG_TRACE
      wfull += clock64() - tw0;
#endif
      const double* ob = ring + size_t(s) * (H::BCH / 8) + (it.kind == 0 ? it.p * 64 : H::NPG * 64);
      if (!DG_SKIPQ(1)) {
        // compile-time shape per item and chunk length: unpredicated DMMAs, loads hoisted
        auto run = [&](auto kcn) {
          constexpr int KCN = decltype(kcn)::value;
          const int kb = c * H::KC;
          if (it.kind == 0) {
            if (it.mc == 1) ho_chunk<N, 0, 1, KCN>(acc, xa, ob, kb, lane);
            if (MU >= 2 && it.mc == 2) ho_chunk<N, 0, (MU >= 2 ? 2 : 1), KCN>(acc, xa, ob, kb, lane);
            if (MU >= 3 && it.mc == 3) ho_chunk<N, 0, (MU >= 3 ? 3 : 1), KCN>(acc, xa, ob, kb, lane);
          } else if (it.kind == 1) {
            if (it.mc == 1) ho_chunk<N, 1, 1, KCN>(acc, xa, ob, kb, lane);
            if (MU >= 2 && it.mc == 2) ho_chunk<N, 1, (MU >= 2 ? 2 : 1), KCN>(acc, xa, ob, kb, lane);
            if (MU >= 3 && it.mc == 3) ho_chunk<N, 1, (MU >= 3 ? 3 : 1), KCN>(acc, xa, ob, kb, lane);
          }
        };
        if (H::KLAST == H::KC || c + 1 < H::NCH) run(std::integral_constant<int, H::KC>{});
        else run(std::integral_constant<int, H::KLAST>{});
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sBar[2 + H::NSLOT + s]);
      __syncwarp();
    }
    gch += H::NCH;
    if (H::SDF && it.kind == 1) {
      // sum the DFMA partials over the 4 lanes of a row; lanes t = 0, 1 take columns 2t, 2t+1
      // (the DMMA accumulator layout the epilogue expects)
#pragma unroll
      for (int m = 0; m < MU; ++m) {
        double sv[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          double v = c < H::GS ? acc[m][c >> 1][c & 1] : 0.0;
          v += __shfl_xor_sync(0xffffffffu, v, 1);
          v += __shfl_xor_sync(0xffffffffu, v, 2);
          sv[c] = v;
        }
        acc[m][0][0] = t4 == 0 ? sv[0] : t4 == 1 ? sv[2] : 0.0;
        acc[m][0][1] = t4 == 0 ? sv[1] : t4 == 1 ? sv[3] : 0.0;
      }
    }
    if (warp == 0) trace_ev(A, j, 7);
#if DG_TRACE
    if (tid == 0 && blockIdx.x == 0 && j < 64 && A.trace) {
      A.trace[j * 16 + 10] = wfull;
      A.trace[j * 16 + 11] = 0;
    }
#endif
    nbar_sync(1, CT);   // every read of X done: it becomes the output staging tile
    if (warp == 0) trace_ev(A, j, 8);
    // ---- epilogue
    const bool staged = MODE == MODE_UPDATE && full;
    double* sres = sX;
    double* sq = sX + EB * 5 * NP;
    if (it.kind >= 0) {
#pragma unroll
      for (int m = 0; m < MU; ++m) {
        if (m >= it.mc) continue;
        const int row = (it.m0 + m) * 8 + g;
        const int e = row / 5, cf = row - 5 * (row / 5);
        if (e >= ne) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (it.kind == 1 && h == 1) continue;
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int n = (it.kind == 0 ? (2 * it.p + h) * 8 : (S::NTL - 1) * 8) + 2 * t4 + q;
            if (n >= NP) continue;
            const int li = row * NP + n;
            const double rhs = acc[m][h][q];
            if (MODE == MODE_UPDATE) {
              const double rr = fma(A.a, rprev[m][h][q], A.dt * rhs);
              const double qn = fma(A.b, rr, q_s[li]);
              if (staged) {
                sres[li] = rr;
                sq[li] = qn;
              } else {
                const size_t gi = size_t(e0) * 5 * NP + li;
                A.res[gi] = rr;
                A.Qout[gi] = qn;
              }
            } else {
              A.out[(size_t(cf) * A.Kpub + A.pub[e0 + e]) * NP + n] = rhs;
            }
          }
        }
      }
    }
    if (warp == 0) trace_ev(A, j, 9);
    if (staged) fence_proxy_async();   // each writer: generic stores before the TMA store reads
    nbar_sync(1, CT);   // staging complete; q_s of this tile no longer read
    if (tid == 0 && staged) {
      fence_proxy_async();
      tma_store_1d(A.res + size_t(e0) * 5 * NP, sres, H::BQ);
      tma_store_1d(A.Qout + size_t(e0) * 5 * NP, sq, H::BQ);
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// ---------------------------------------------------------------- modal-quadrature scheme (N3)
// The paper's own discretisation (Appendix A; reading A23):
// unknowns are coefficients of the orthonormal basis psi, the weak form is integrated by
// collapsed Gauss-Jacobi rules with p+1 points per direction (degree 2p+1) on the tet and on
// each face, every face at the points of its owner (smaller global element id):
//   dc_i/dt = sum_q w_q sum_a dpsi_i/dxi_a(q) Ft_a(u(q)) - sum_f Fscale_f sum_q w^f_q psi_i(q) F*_n(q).
// Tables (ModalTables, concatenated; MS<P> offsets) are read through the L1.
template <int P>
struct MS {
  static constexpr int NP = (P + 1) * (P + 2) * (P + 3) / 6, NQ1 = P + 1;
  static constexpr int NQ = NQ1 * NQ1 * NQ1, NQF = NQ1 * NQ1;
  // table offsets (doubles) in the concatenation of refelem.h ModalTables
  static constexpr int O_WQ = 0, O_VQ = O_WQ + NQ, O_DQ = O_VQ + NQ * NP, O_WF = O_DQ + 3 * NP * NQ;
  static constexpr int O_PSTD = O_WF + NQF, O_PMAP = O_PSTD + 4 * NQF * NP, O_V = O_PMAP + 96 * NQF * NP;
  static constexpr int O_VINV = O_V + NP * NP, TOTAL = O_VINV + NP * NP;
};

// Each warp owns one element at a time (persistent CTAs, warps stride over the elements), its coefficients, its
// neighbours' coefficients and its quadrature values in a private slice of shared memory;
// lanes map to quadrature points for the interpolations and fluxes and to (field, mode)
// pairs for the projections; only __syncwarp between the steps.
template <int P>
struct MW {
  using M = MS<P>;
  static constexpr int NP = M::NP, NQ = M::NQ, NQF = M::NQF;
  static constexpr int EPW = NQ <= 8 ? 4 : 1;                          // elements per warp
  static constexpr int WPC = P <= 2 ? 8 : 4, NT = 32 * WPC;           // warps per CTA
  static constexpr int MINB = P <= 2 ? 2 : 1;                          // CTAs per SM (register cap)
  // one element's slice: coefficients, neighbours' coefficients, volume fluxes, wave speeds,
  // weighted face fluxes
  static constexpr int E_C = 0, E_CN = E_C + 5 * NP, E_FV = E_CN + 4 * 5 * NP, E_LAM = E_FV + 15 * NQ,
                       E_FS = E_LAM + 4 * NQF, E_END = E_FS + 5 * 4 * NQF;
  static constexpr int ESTRIDE = E_END | 1;                            // odd: element-parallel reads
  static constexpr int WSTRIDE = EPW * ESTRIDE;
  static constexpr size_t SMEM = size_t(WPC) * WSTRIDE * 8 + size_t(WPC) * EPW * 4 * 4;
};

// Each warp owns EPW elements at a time (persistent CTAs, warps stride over element groups),
// their coefficients, their neighbours' coefficients and their quadrature values in a private
// slice of shared memory; lanes map to (element, quadrature point) for the interpolations and
// fluxes and to (element, field, mode) for the projections; only __syncwarp between steps.
template <int P, int MODE>
__global__ void __launch_bounds__(MW<P>::NT, MW<P>::MINB) modal_warp_kernel(const StageArgs A) {
  using M = MS<P>;
  using W = MW<P>;
  constexpr int NP = M::NP, NQ = M::NQ, NQF = M::NQF, EPW = W::EPW, ES = W::ESTRIDE;
  extern __shared__ __align__(16) double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* ws = sm + warp * W::WSTRIDE;
  int* own_s = reinterpret_cast<int*>(sm + W::WPC * W::WSTRIDE) + warp * EPW * 4;   // [EPW][4]
  const double* T = A.op;
  const double gamma = A.gamma, gm1 = A.gamma - 1.0;
  const int nel = A.e_end - A.e_begin;
  for (int g0 = (blockIdx.x * W::WPC + warp) * EPW; g0 < nel; g0 += gridDim.x * W::WPC * EPW) {
    const int ne = min(EPW, nel - g0);
    const int k0 = A.e_begin + g0;
    for (int i = lane; i < ne * 5 * NP; i += 32) {
      const int ee = i / (5 * NP), r0 = i - ee * 5 * NP;
      ws[ee * ES + W::E_C + r0] = A.Qin[size_t(k0 + ee) * 5 * NP + r0];
    }
    for (int i = lane; i < ne * 4 * 5 * NP; i += 32) {
      const int ee = i / (20 * NP), r1 = i - ee * 20 * NP, f = r1 / (5 * NP), r0 = r1 - f * 5 * NP;
      const int k = k0 + ee;
      const int code = A.code[size_t(k) * 4 + f];
      ws[ee * ES + W::E_CN + r1] =
          code < CODE_GHOST ? __ldg(A.Qin + size_t(A.nbr[size_t(k) * 4 + f]) * 5 * NP + r0) : 0.0;
    }
    __syncwarp();
    // ---- volume points: values, validity, contravariant fluxes
    for (int v = lane; v < ne * NQ; v += 32) {
      const int ee = v / NQ, q = v - ee * NQ;
      const int k = k0 + ee;
      const double* c_s = ws + ee * ES + W::E_C;
      const double* G = A.geo + size_t(k) * GEO;
      double u[5];
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        double acc = 0;
        for (int i = 0; i < NP; ++i) acc = fma(__ldg(T + M::O_VQ + q * NP + i), c_s[c * NP + i], acc);
        u[c] = acc;
      }
      const double ri = 1.0 / u[0];
      const double vx = u[1] * ri, vy = u[2] * ri, vz = u[3] * ri;
      const double p = gm1 * (u[4] - 0.5 * (u[1] * vx + u[2] * vy + u[3] * vz));
      if (!state_ok(u[0], p, u[1], u[2], u[3], u[4])) flag_blowup(A.flag, A.gid[k]);
      const double pd = p - A.pref, Ep = u[4] + p;
      double* fv_s = ws + ee * ES + W::E_FV;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double cx = G[3 * a], cy = G[3 * a + 1], cz = G[3 * a + 2];
        const double U = cx * vx + cy * vy + cz * vz;
        double* o = fv_s + (a * 5) * NQ + q;
        o[0] = u[0] * U;
        o[NQ] = fma(cx, pd, u[1] * U);
        o[2 * NQ] = fma(cy, pd, u[2] * U);
        o[3 * NQ] = fma(cz, pd, u[3] * U);
        o[4 * NQ] = Ep * U;
      }
    }
    // ---- face points: both traces at the owner's points; each lane keeps the traces of its
    //      (at most FR) points for the flux pass after the face max
    constexpr int FR = (EPW * 4 * NQF + 31) / 32;
    double um[FR][5], up[FR][5];
#pragma unroll
    for (int rr = 0; rr < FR; ++rr) {
      const int v = lane + 32 * rr;
      if (v >= ne * 4 * NQF) break;
      const int ee = v / (4 * NQF), fq = v - ee * 4 * NQF, f = fq / NQF, q = fq - f * NQF;
      const int k = k0 + ee;
      const double* c_s = ws + ee * ES + W::E_C;
      const double* cn_s = ws + ee * ES + W::E_CN;
      const int code = A.code[size_t(k) * 4 + f], nb = A.nbr[size_t(k) * 4 + f];
      const double* Gf = A.geo + size_t(k) * GEO + 9 + 4 * f;
      int own_off = M::O_PSTD + f * NQF * NP, nb_off = 0;
      if (code < CODE_GHOST) {
        const int f2 = code / 6, sg = code - 6 * f2;
        if (A.gid[k] < A.gid[nb]) {
          nb_off = M::O_PMAP + ((f * 4 + f2) * 6 + sg) * NQF * NP;
        } else {
          own_off = M::O_PMAP + ((f2 * 4 + f) * 6 + PERM_INV[sg]) * NQF * NP;
          nb_off = M::O_PSTD + f2 * NQF * NP;
        }
      }
      if (q == 0) own_s[ee * 4 + f] = own_off;
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        double acc = 0;
        for (int i = 0; i < NP; ++i) acc = fma(__ldg(T + own_off + q * NP + i), c_s[c * NP + i], acc);
        um[rr][c] = acc;
      }
      if (code < CODE_GHOST) {
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          double acc = 0;
          for (int i = 0; i < NP; ++i) acc = fma(__ldg(T + nb_off + q * NP + i), cn_s[(f * 5 + c) * NP + i], acc);
          up[rr][c] = acc;
        }
      } else {
        ghost_trace(A, code - CODE_BC, um[rr], Gf[0], Gf[1], Gf[2], up[rr]);
      }
      auto speed = [&](const double (&w)[5]) {
        const double ri = 1.0 / w[0];
        const double un = (w[1] * Gf[0] + w[2] * Gf[1] + w[3] * Gf[2]) * ri;
        const double p = gm1 * (w[4] - 0.5 * (w[1] * w[1] + w[2] * w[2] + w[3] * w[3]) * ri);
        return fabs(un) + sqrt(gamma * p * ri);
      };
      ws[ee * ES + W::E_LAM + fq] = fmax(speed(um[rr]), speed(up[rr]));
    }
    __syncwarp();
#pragma unroll
    for (int rr = 0; rr < FR; ++rr) {
      const int v = lane + 32 * rr;
      if (v >= ne * 4 * NQF) break;
      const int ee = v / (4 * NQF), fq = v - ee * 4 * NQF, f = fq / NQF, q = fq - f * NQF;
      const double* Gf = A.geo + size_t(k0 + ee) * GEO + 9 + 4 * f;
      const double nx = Gf[0], ny = Gf[1], nz = Gf[2];
      const double* lam_s = ws + ee * ES + W::E_LAM;
      double lam = lam_s[fq];
      if (A.lambda_mode == 0)
        for (int qq = 0; qq < NQF; ++qq) lam = fmax(lam, lam_s[f * NQF + qq]);
      auto nflux = [&](const double (&w)[5], double* fo) {
        const double ri = 1.0 / w[0];
        const double un = (w[1] * nx + w[2] * ny + w[3] * nz) * ri;
        const double p = gm1 * (w[4] - 0.5 * (w[1] * w[1] + w[2] * w[2] + w[3] * w[3]) * ri);
        const double pd = p - A.pref;
        fo[0] = w[0] * un;
        fo[1] = fma(pd, nx, w[1] * un);
        fo[2] = fma(pd, ny, w[2] * un);
        fo[3] = fma(pd, nz, w[3] * un);
        fo[4] = (w[4] + p) * un;
      };
      double fm[5], fp[5];
      nflux(um[rr], fm);
      nflux(up[rr], fp);
      const double sc = Gf[3] * __ldg(T + M::O_WF + q);
      double* fs_s = ws + ee * ES + W::E_FS;
#pragma unroll
      for (int c = 0; c < 5; ++c)
        fs_s[c * 4 * NQF + fq] = sc * (0.5 * (fm[c] + fp[c]) - 0.5 * lam * (up[rr][c] - um[rr][c]));
    }
    __syncwarp();
    // ---- projection onto the basis, update (or rhs out as nodal values)
    constexpr int PR = (EPW * 5 * NP + 31) / 32;
    double rhs[PR];
#pragma unroll
    for (int rr = 0; rr < PR; ++rr) {
      const int v = lane + 32 * rr;
      rhs[rr] = 0.0;
      if (v >= ne * 5 * NP) break;
      const int ee = v / (5 * NP), ci = v - ee * 5 * NP, c = ci / NP, i = ci - c * NP;
      const int k = k0 + ee;
      const double* fv_s = ws + ee * ES + W::E_FV;
      const double* fs_s = ws + ee * ES + W::E_FS;
      // four interleaved partial sums: the 3 NQ + 4 NQF long dot product is a latency chain
      double acc4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double* D = T + M::O_DQ + (a * NP + i) * NQ;
        const double* F = fv_s + (a * 5 + c) * NQ;
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc4[(a * NQ + q) & 3] = fma(__ldg(D + q), F[q], acc4[(a * NQ + q) & 3]);
      }
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        const double* Pt = T + own_s[ee * 4 + f];
        const double* F = fs_s + c * 4 * NQF + f * NQF;
#pragma unroll
        for (int q = 0; q < NQF; ++q) acc4[(f * NQF + q) & 3] = fma(-__ldg(Pt + q * NP + i), F[q], acc4[(f * NQF + q) & 3]);
      }
      const double acc = (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
      rhs[rr] = acc;
      if (MODE == MODE_UPDATE) {
        const size_t gi = size_t(k) * 5 * NP + ci;
        const double r2 = fma(A.a, A.res[gi], A.dt * acc);
        A.res[gi] = r2;
        A.Qout[gi] = fma(A.b, r2, ws[ee * ES + W::E_C + ci]);
      }
    }
    if (MODE == MODE_RHS) {   // V (dc/dt) into the public layout, staged in the volume-flux slice
      __syncwarp();
#pragma unroll
      for (int rr = 0; rr < PR; ++rr) {
        const int v = lane + 32 * rr;
        if (v < ne * 5 * NP) {
          const int ee = v / (5 * NP), ci = v - ee * 5 * NP;
          ws[ee * ES + W::E_FV + ci] = rhs[rr];
        }
      }
      __syncwarp();
      for (int v = lane; v < ne * 5 * NP; v += 32) {
        const int ee = v / (5 * NP), cn = v - ee * 5 * NP, c = cn / NP, n = cn - c * NP;
        const double* r_s = ws + ee * ES + W::E_FV;
        double acc = 0;
        for (int i = 0; i < NP; ++i) acc = fma(__ldg(T + M::O_V + n * NP + i), r_s[c * NP + i], acc);
        A.out[(size_t(c) * A.Kpub + A.pub[k0 + ee]) * NP + n] = acc;
      }
    }
    __syncwarp();   // the warp's slice is reused by its next element group
  }
}

// nodal values <-> modal coefficients per element and field: out = Mat (NP x NP) in
__global__ void modal_convert_kernel(const double* __restrict__ in, double* __restrict__ out,
                                     const double* __restrict__ Mat, int64_t K, int NP) {
  const int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (idx >= K * 5 * NP) return;
  const int64_t row = idx / NP;
  const int n = int(idx - row * NP);
  const double* x = in + row * NP;
  double acc = 0;
  for (int i = 0; i < NP; ++i) acc = fma(Mat[n * NP + i], x[i], acc);
  out[idx] = acc;
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

// point sensors: one warp per sensor interpolates the five conserved
// variables with the host-computed nodal weights, then forms p from them; NaN rows for
// sensors that are not on this rank
__global__ void sensor_kernel(const double* __restrict__ Q, const int32_t* __restrict__ el,
                              const double* __restrict__ w, int n, int Np, double gamma, double* __restrict__ out) {
  const int sid = int((blockIdx.x * size_t(blockDim.x) + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (sid >= n) return;
  double* o = out + size_t(sid) * 6;
  const int k = el[sid];
  if (k < 0) {
    if (lane < 6) o[lane] = __longlong_as_double(0x7ff8000000000000LL);
    return;
  }
  double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int j = lane; j < Np; j += 32) {
    const double wj = w[size_t(sid) * Np + j];
#pragma unroll
    for (int c = 0; c < 5; ++c) acc[c] = fma(wj, Q[(size_t(k) * 5 + c) * Np + j], acc[c]);
  }
#pragma unroll
  for (int c = 0; c < 5; ++c)
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], d);
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < 5; ++c) o[c] = acc[c];
    o[5] = (gamma - 1.0) * (acc[4] - 0.5 * (acc[1] * acc[1] + acc[2] * acc[2] + acc[3] * acc[3]) / acc[0]);
  }
}

}  // namespace dgk
