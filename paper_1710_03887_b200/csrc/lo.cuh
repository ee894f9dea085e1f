// sm_100a stage kernels for the paper's own order (the paper runs p = 1): the
// nodal scheme at N = 1 (stage_lo4_kernel) and the paper's modal-quadrature scheme at p = 1
// (modal_lo4_kernel) -- the same fused RK stage as stage_ws_kernel / modal_tile_kernel (volume
// flux Eq. 1-2; traces and ghosts Eqs. 3-7; LLF flux; LSERK update),
// laid out for what bounds this order: at N = 1 a stage is 2,940 flop against 864 compulsory
// bytes per element (3.4 flop/B, ridge 5.7), i.e. HBM-bound, and the operators are 4 x 4 -- too
// small for the DMMA tiling of the N >= 2 kernels, whose per-tile barriers and fragment traffic
// dominated here (36 GDOF/s, 0.24 of the HBM roofline).  Four lanes per element, tiles streamed
// by TMA through three shared-memory buffers with a dedicated IO warp, no barrier between compute
// warps.  (A one-thread-per-element version with the operator as constant-bank immediates
// measured 54 GDOF/s at N = 1 -- latency-bound: shared memory fixes the elements in flight -- and
// 21 at N = 2 (spills); it is in the git history of round 2.)
// Per-element arithmetic does not depend on tile, CTA or partition (bitwise partition
// invariance holds as for the other kernels).
#pragma once
#include "kernels.cuh"

namespace dgk {

// kernel-parameter operator (constant bank): v[k * 4 + n] = Op[n][k], k < 12: -Dr, -Ds, -Dt; then LIFT
template <int N>
struct LoOp {
  static_assert(N == 1, "the four-lane kernel is the N = 1 kernel");
  double v[24 * 4];
  int fm[12];
};

// ---------------------------------------------------------------- N = 1, four lanes per element
// At N = 1 an element has Np = 4 nodes and 4 faces of Nfp = 3 nodes: lane (e, n) of a warp
// (8 elements x 4 lanes) computes the volume flux of node n and node n of EACH face (lane 3 rides
// along on node 0's addresses; its face results meet zero LIFT columns), applies its OWN columns
// of Op = [-Dr -Ds -Dt LIFT] to them (partial sums for all four output nodes, 120 FMAs, the
// columns read as 16-byte shared-memory broadcasts), and the element's four lanes sum their
// partials with a transposing butterfly (xor 1, xor 2: 15 64-bit shuffles) that leaves output
// node n on lane n.  The kernel's elements in flight are set by shared memory (540 B per element
// and buffer), so what counts is the latency per element: four lanes cut it to about a quarter
// of one thread per element (54 -> 76 GDOF/s), the three lanes of a face reading ONE 32-byte
// sector of the neighbour per field cut the gathers' L1 wavefronts from 48 to 16 per element
// (-> 87), and gathering one face ahead freed the registers that spilled (-> 92).
// Tiles of T = 120 elements in THREE buffers: the IO warp stores tile j, waits for the store's
// shared-memory reads and refills the buffer with tile j + 3 while the 15 compute warps work
// through tiles j + 1 and j + 2; compute warps never wait for each other.  16 warps in all: 128
// registers per thread (a 17th warp would put five on one scheduler: 96 registers, spills).
struct LO4 {
  static constexpr int NP = 4, NFP = 3, KT = 28;   // per-lane operator columns: 12 volume + 16 face
#ifdef DG_LO4_T
  static constexpr int T = DG_LO4_T;
#else
  static constexpr int T = 120;   // 15 compute warps + the IO warp = 16 warps: 128 registers per thread
#endif
  static constexpr int NB = 3;                                // tile buffers
  static constexpr int CT = 4 * T, NT = CT + 32;              // compute threads + the IO warp
  static_assert(T % 8 == 0 && NT <= 1024, "whole warps of 8 elements; tile addresses stay 16-byte aligned");
  static constexpr uint32_t BQ = uint32_t(T) * 5 * NP * 8;
  static constexpr uint32_t BG = uint32_t(T) * GEO * 8;
  static constexpr uint32_t BN = uint32_t(T) * 16;
  static constexpr uint32_t BC = uint32_t(T) * 4;
  static constexpr uint32_t BUF = 2 * BQ + BG + BN + BC;      // Q | res | geo | nbr | code
  static constexpr size_t SMEM_OP = 4 * KT * 8;               // [lane n][24] operator columns
  static constexpr size_t SMEM_T = size_t(2 * 96 * NFP + 15) / 16 * 16;
  static constexpr size_t SMEM = NB * size_t(BUF) + SMEM_OP + SMEM_T + 32 + 80;   // + barriers + ghost states
  static_assert(SMEM <= 227 * 1024, "tile buffers do not fit in shared memory");
};

template <int MODE>
__global__ void __launch_bounds__(LO4::NT, 1) stage_lo4_kernel(const StageArgs A, const LoOp<1> O) {
  using L = LO4;
  constexpr int NP = 4, NFP = 3, T = L::T, NT = L::NT, NB = L::NB;
  extern __shared__ __align__(128) unsigned char smem[];
  auto bufQ = [&](int b) { return reinterpret_cast<double*>(smem + size_t(b) * L::BUF); };
  auto bufR = [&](int b) { return reinterpret_cast<double*>(smem + size_t(b) * L::BUF + L::BQ); };
  auto bufG = [&](int b) { return reinterpret_cast<double*>(smem + size_t(b) * L::BUF + 2 * L::BQ); };
  auto bufN = [&](int b) { return reinterpret_cast<int*>(smem + size_t(b) * L::BUF + 2 * L::BQ + L::BG); };
  auto bufC = [&](int b) { return reinterpret_cast<uint8_t*>(smem + size_t(b) * L::BUF + 2 * L::BQ + L::BG + L::BN); };
  double* sOp = reinterpret_cast<double*>(smem + NB * size_t(L::BUF));
  uint8_t* sTbl = reinterpret_cast<uint8_t*>(sOp) + L::SMEM_OP;
  uint8_t* sTblf = sTbl + 96 * NFP;
  uint64_t* sBar = reinterpret_cast<uint64_t*>(sTbl + L::SMEM_T);   // full[NB]
  // ghost states that do not depend on the interior trace: [0] pass-through (Eq. 3), [1] inflow
  // at this stage's time (Eqs. 5-7: pow and cos evaluated once per CTA, not per face node)
  double* sGh = reinterpret_cast<double*>(sBar + 4);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if ((DG_PDL >> 1) & 1) pdl_launch_dependents();
  for (int i = tid; i < 96 * NFP; i += NT) {
    sTbl[i] = A.tbl[i];
    sTblf[i] = A.tblf[i];
  }
  // lane n's operator columns: [d][nn] = Op[nn][4 d + n] (its volume node), then [f][nn] =
  // LIFT[nn][3 f + n] (its node of face f; zero for lane 3, which has no face node)
  if (tid < 4 * L::KT) {
    const int n = tid / L::KT, k = tid % L::KT, nn = k & 3;
    if (k < 12) sOp[tid] = O.v[((k >> 2) * 4 + n) * 4 + nn];
    else if (k < 28) sOp[tid] = n < NFP ? O.v[(12 + 3 * ((k - 12) >> 2) + n) * 4 + nn] : 0.0;
  }
  if (tid == 0)
    for (int b = 0; b < NB; ++b) mbar_init(&sBar[b], 1);
  if (tid == 32) {
    double qi[5];
    inflow_state(A, qi);
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      sGh[c] = A.qinf[c];
      sGh[5 + c] = qi[c];
    }
  }
  __syncthreads();
  if ((DG_PDL >> 1) & 1) pdl_wait();
  const int ntiles = (A.e_end - A.e_begin + T - 1) / T;
  const int nmine = (ntiles > (int)blockIdx.x) ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  auto tile_e0 = [&](int jj) { return A.e_begin + (int(blockIdx.x) + jj * int(gridDim.x)) * T; };
  auto tile_full = [&](int jj) { return A.e_end - tile_e0(jj) >= T; };
  constexpr int BAR_DONE = 1;   // named barriers 1 .. NB: buffer b's tile computed

  if (warp == L::CT / 32) {
    // ======================= IO warp
    auto issue_load = [&](int jj) {   // lane 0; the buffer's previous bulk stores have been read
      const int b = jj % NB;
      if (tile_full(jj)) {
        const size_t e0 = size_t(tile_e0(jj));
        fence_proxy_async();
        mbar_arrive_expect_tx(&sBar[b], (MODE == MODE_UPDATE ? 2 * L::BQ : L::BQ) + L::BG + L::BN + L::BC);
        tma_load_1d(bufQ(b), A.Qin + e0 * 5 * NP, L::BQ, &sBar[b]);
        if (MODE == MODE_UPDATE) tma_load_1d(bufR(b), A.res + e0 * 5 * NP, L::BQ, &sBar[b]);
        tma_load_1d(bufG(b), A.geo + e0 * GEO, L::BG, &sBar[b]);
        tma_load_1d(bufN(b), A.nbr + e0 * 4, L::BN, &sBar[b]);
        tma_load_1d(bufC(b), A.code + e0 * 4, L::BC, &sBar[b]);
      } else {
        // the partial last tile: its lanes fill their slots with plain loads; hand the buffer over
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&sBar[b])) : "memory");
      }
    };
    if (lane == 0)
      for (int jj = 0; jj < NB && jj < nmine; ++jj) issue_load(jj);
    for (int j = 0; j < nmine; ++j) {
      const int b = j % NB;
      nbar_sync(BAR_DONE + b, NT);
      if (lane == 0) {
        const bool st = MODE == MODE_UPDATE && tile_full(j);
        if (st) {
          const size_t e0 = size_t(tile_e0(j));
          fence_proxy_async();
          tma_store_1d(A.Qout + e0 * 5 * NP, bufQ(b), L::BQ);
          tma_store_1d(A.res + e0 * 5 * NP, bufR(b), L::BQ);
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
        if (j + NB < nmine) {
          if (st) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
          issue_load(j + NB);
        }
      }
      __syncwarp();
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    return;
  }

  // ======================= compute warps: lane (es, n) = element slot es of the tile, node / face n
  const double gamma = A.gamma, gm1 = A.gamma - 1.0;
  const int es = tid >> 2, n = tid & 3;
  const int ii = n < NFP ? n : 0;   // face node of this lane (lane 3: node 0 again, zero LIFT columns)
  const int fm0 = A.fmask[ii], fm1 = A.fmask[NFP + ii], fm2 = A.fmask[2 * NFP + ii], fm3 = A.fmask[3 * NFP + ii];
  const double* cf = sOp + n * L::KT;
  const bool o1 = n & 1, o2 = (n & 2) != 0;
  for (int j = 0; j < nmine; ++j) {
    const int b = j % NB;
    const int e0 = tile_e0(j);
    const int ne = min(T, A.e_end - e0);
    const bool full = ne == T;
    double* q_s = bufQ(b) + es * 5 * NP;
    double* r_s = bufR(b) + es * 5 * NP;
    double* g_s = bufG(b) + es * GEO;
    int* n_s = bufN(b) + es * 4;
    uint8_t* c_s = bufC(b) + es * 4;
    mbar_wait(&sBar[b], (j / NB) & 1);
    const bool active = es < ne;
    // slots past a partial tile's elements work on its last element and store nothing
    const size_t eg = size_t(e0) + (active ? es : ne - 1);
    if (!full) {
#pragma unroll
      for (int c = 0; c < 5; ++c) q_s[c * NP + n] = __ldg(A.Qin + eg * 5 * NP + c * NP + n);
      for (int i = n; i < GEO; i += 4) g_s[i] = __ldg(A.geo + eg * GEO + i);
      n_s[n] = __ldg(A.nbr + eg * 4 + n);
      c_s[n] = A.code[eg * 4 + n];
      __syncwarp();
    }
    // ---- neighbour traces (issued first: the latency hides behind the volume node).  Lane i of
    //      the element gathers node i of ALL four faces, so the three lanes of a face read one
    //      32-byte sector of the neighbour (one row of 4 nodes) in one wavefront per field; lane 3
    //      rides along on node 0's addresses and its face results are weighted by zero columns
#ifndef DG_LO4_LA
#define DG_LO4_LA 1
#endif
    double qp[DG_LO4_LA ? 1 : 4][5];
    int tagf[4];
    const double* qsrc[4];
    int qstr[4];
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const int code = c_s[f], nb = n_s[f];
      tagf[f] = code >= CODE_BC ? code - CODE_BC : 0;
      qsrc[f] = code < CODE_GHOST ? A.Qin + size_t(nb) * 5 * NP + sTbl[(f * 24 + code) * NFP + ii]
                : code < CODE_BC ? A.recv + size_t(nb) * 5 * NFP + sTblf[(f * 24 + code - CODE_GHOST) * NFP + ii] : A.Qin;
      qstr[f] = code < CODE_GHOST ? NP : code < CODE_BC ? NFP : 0;
    }
    // face 0 now (behind the volume node), face f + 1 while face f is computed; boundary faces
    // read a dummy (the first state row) that the ghost below overwrites
    auto gather = [&](int f, double (&dst)[5]) {
#pragma unroll
      for (int c = 0; c < 5; ++c) dst[c] = __ldg(qsrc[f] + c * qstr[f]);
    };
    if (DG_LO4_LA) gather(0, qp[0]);
    else {
#pragma unroll
      for (int f = 0; f < 4; ++f) gather(f, qp[f]);
    }
    // ---- volume node n: contravariant fluxes times this lane's columns of -Dr, -Ds, -Dt
    double part[5][NP];
    {
      const double rho = q_s[n], mx = q_s[NP + n], my = q_s[2 * NP + n], mz = q_s[3 * NP + n], E = q_s[4 * NP + n];
      const double ri = rcp_nr(rho);
      const double u = mx * ri, v = my * ri, w = mz * ri;
      const double p = gm1 * (E - 0.5 * (mx * u + my * v + mz * w));
      if (active && !state_ok(rho, p, mx, my, mz, E)) flag_blowup(A.flag, A.gid[eg]);
      const double Ep = E + p, pd = p - A.pref;   // background-flux subtraction (A14)
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double cx = g_s[3 * d], cy = g_s[3 * d + 1], cz = g_s[3 * d + 2];
        const double U = cx * u + cy * v + cz * w;
        double fl[5];
        fl[0] = rho * U;
        fl[1] = fma(cx, pd, mx * U);
        fl[2] = fma(cy, pd, my * U);
        fl[3] = fma(cz, pd, mz * U);
        fl[4] = Ep * U;
        const double2 c01 = *reinterpret_cast<const double2*>(cf + 4 * d);
        const double2 c23 = *reinterpret_cast<const double2*>(cf + 4 * d + 2);
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          part[c][0] = d == 0 ? c01.x * fl[c] : fma(c01.x, fl[c], part[c][0]);
          part[c][1] = d == 0 ? c01.y * fl[c] : fma(c01.y, fl[c], part[c][1]);
          part[c][2] = d == 0 ? c23.x * fl[c] : fma(c23.x, fl[c], part[c][2]);
          part[c][3] = d == 0 ? c23.y * fl[c] : fma(c23.y, fl[c], part[c][3]);
        }
      }
    }
    // ---- faces: node i of each face on lane i; LLF flux with the face maximum of the wave
    //      speed (max over the element's lanes: two shuffles), times this lane's LIFT columns
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const double nx = g_s[9 + 4 * f], ny = g_s[9 + 4 * f + 1], nz = g_s[9 + 4 * f + 2];
      const double hfs = 0.5 * g_s[9 + 4 * f + 3];
      const int fm = f == 0 ? fm0 : f == 1 ? fm1 : f == 2 ? fm2 : fm3;
      double qq[5];
#pragma unroll
      for (int c = 0; c < 5; ++c) qq[c] = qp[DG_LO4_LA ? 0 : f][c];
      if (DG_LO4_LA && f < 3) gather(f + 1, qp[0]);
      const double qm0 = q_s[fm], qm1 = q_s[NP + fm], qm2 = q_s[2 * NP + fm], qm3 = q_s[3 * NP + fm], qm4 = q_s[4 * NP + fm];
      if (tagf[f] == 1) {          // slip wall: mirror the normal momentum (Eq. 4)
        const double mn = qm1 * nx + qm2 * ny + qm3 * nz;
        qq[0] = qm0;
        qq[1] = qm1 - 2.0 * mn * nx;
        qq[2] = qm2 - 2.0 * mn * ny;
        qq[3] = qm3 - 2.0 * mn * nz;
        qq[4] = qm4;
      } else if (tagf[f]) {        // pass-through (2) / inflow (3)
        const double* gh = sGh + (tagf[f] == 2 ? 0 : 5);
#pragma unroll
        for (int c = 0; c < 5; ++c) qq[c] = gh[c];
      }
      const double rim = rcp_nr(qm0);
      const double unm = (qm1 * nx + qm2 * ny + qm3 * nz) * rim;
      const double pm = gm1 * (qm4 - 0.5 * (qm1 * qm1 + qm2 * qm2 + qm3 * qm3) * rim);
      const double rip = rcp_nr(qq[0]);
      const double unp = (qq[1] * nx + qq[2] * ny + qq[3] * nz) * rip;
      const double pp = gm1 * (qq[4] - 0.5 * (qq[1] * qq[1] + qq[2] * qq[2] + qq[3] * qq[3]) * rip);
      double lam = fmax(fabs(unm) + sqrt_nr(gamma * pm * rim), fabs(unp) + sqrt_nr(gamma * pp * rip));
      const double dp = pm - pp;
      double gf[5], dq[5];
      gf[0] = fma(qm0, unm, -qq[0] * unp);
      gf[1] = fma(dp, nx, fma(qm1, unm, -qq[1] * unp));
      gf[2] = fma(dp, ny, fma(qm2, unm, -qq[2] * unp));
      gf[3] = fma(dp, nz, fma(qm3, unm, -qq[3] * unp));
      gf[4] = fma(qm4 + pm, unm, -(qq[4] + pp) * unp);
      dq[0] = qq[0] - qm0;
      dq[1] = qq[1] - qm1;
      dq[2] = qq[2] - qm2;
      dq[3] = qq[3] - qm3;
      dq[4] = qq[4] - qm4;
      if (A.lambda_mode == 0) {    // positive doubles order like their bit patterns
        long long a = __double_as_longlong(lam);
        long long o = __shfl_xor_sync(0xffffffffu, a, 1);
        a = a > o ? a : o;
        o = __shfl_xor_sync(0xffffffffu, a, 2);
        lam = __longlong_as_double(a > o ? a : o);
      }
      const double2 c01 = *reinterpret_cast<const double2*>(cf + 12 + 4 * f);
      const double2 c23 = *reinterpret_cast<const double2*>(cf + 12 + 4 * f + 2);
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        const double dF = hfs * fma(lam, dq[c], gf[c]);
        part[c][0] = fma(c01.x, dF, part[c][0]);
        part[c][1] = fma(c01.y, dF, part[c][1]);
        part[c][2] = fma(c23.x, dF, part[c][2]);
        part[c][3] = fma(c23.y, dF, part[c][3]);
      }
    }
    // ---- sum the four lanes' partials; lane n keeps output node n (transposing butterfly)
    double rhs[5];
    {
      double k0[5], k1[5];
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        const double s0 = __shfl_xor_sync(0xffffffffu, o1 ? part[c][0] : part[c][1], 1);
        const double s1 = __shfl_xor_sync(0xffffffffu, o1 ? part[c][2] : part[c][3], 1);
        k0[c] = (o1 ? part[c][1] : part[c][0]) + s0;   // node o1
        k1[c] = (o1 ? part[c][3] : part[c][2]) + s1;   // node 2 + o1
      }
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        const double s = __shfl_xor_sync(0xffffffffu, o2 ? k0[c] : k1[c], 2);
        rhs[c] = (o2 ? k1[c] : k0[c]) + s;             // node 2 o2 + o1 = n
      }
    }
    // ---- LSERK update in place in the tile (full tiles), or straight to global memory
    if (MODE == MODE_UPDATE) {
      if (full) {
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          const double rr = fma(A.a, r_s[c * NP + n], A.dt * rhs[c]);
          const double qo = q_s[c * NP + n];
          r_s[c * NP + n] = rr;
          // every lane of the element has read the element's Q for its face by now only if the
          // four lanes are past their face phase: they are (the butterfly's shuffles are warp-wide)
          q_s[c * NP + n] = fma(A.b, rr, qo);
        }
      } else if (active) {
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          const size_t gi = eg * 5 * NP + c * NP + n;
          const double rr = fma(A.a, __ldg(A.res + gi), A.dt * rhs[c]);
          A.res[gi] = rr;
          A.Qout[gi] = fma(A.b, rr, q_s[c * NP + n]);
        }
      }
    } else if (active) {
      const size_t pe = size_t(A.pub[eg]);
#pragma unroll
      for (int c = 0; c < 5; ++c) A.out[(size_t(c) * A.Kpub + pe) * NP + n] = rhs[c];
    }
    // order this thread's generic-proxy tile writes before the IO warp's bulk stores
    if (MODE == MODE_UPDATE && full) fence_proxy_async();
    nbar_arrive(BAR_DONE + b, NT);
  }
}

}  // namespace dgk

namespace dgk {

// ---------------------------------------------------------------- the paper's scheme at the paper's order
// Modal-quadrature scheme at p = 1 ("p = 1", Appendix A; DESIGN.md reading
// A23; same arithmetic as modal_tile_kernel, modal.cuh): Np = 4 modes, (p+1)^3 = 8 volume points,
// (p+1)^2 = 4 points per face -- again four lanes per element on the stage_lo4_kernel frame
// (three TMA tile buffers of 120 elements, IO warp, no barrier between compute warps):
//   lane n: volume points n and n + 4 (values by 4-term sums, contravariant fluxes, projected at
//           once onto all four modes with the point's w dpsi/dxi columns);
//           point n of each face: own trace with the face's table row of this point, neighbour
//           trace from the neighbour's coefficients -- lane n gathers mode n of the five fields
//           (the element's four lanes read one 32-byte sector per field), the 20 values are
//           exchanged through a per-warp scratch slot -- ghosts, wave speed, face max by two
//           shuffles, LLF flux times Fscale w, projected with the same table row;
//   the four lanes' partial dc/dt are summed by the transposing butterfly, lane n keeps mode n,
//   and the LSERK update is done in place in the tile.
struct ML4 {
  using M = MS<1>;
  static constexpr int NP = 4, NQ = 8, NQF = 4;
#ifdef DG_ML4_T
  static constexpr int T = DG_ML4_T;
#else
  static constexpr int T = 120;
#endif
  static constexpr int NB = 3;
  static constexpr int CT = 4 * T, NT = CT + 32;
  static_assert(T % 8 == 0 && NT <= 1024, "whole warps of 8 elements; tile addresses stay 16-byte aligned");
  static constexpr uint32_t BQ = uint32_t(T) * 5 * NP * 8;
  static constexpr uint32_t BG = uint32_t(T) * GEO * 8;
  static constexpr uint32_t BN = uint32_t(T) * 16;
  static constexpr uint32_t BC = uint32_t(T) * 4;
  static constexpr uint32_t BM = uint32_t(T) * 8;
  static constexpr uint32_t BUF = 2 * BQ + BG + BN + BC + BM;   // coefficients | res | geo | nbr | code | table ids
  static_assert(BQ % 16 == 0 && BG % 16 == 0 && BN % 16 == 0 && BC % 16 == 0 && BM % 16 == 0, "TMA sizes");
  static constexpr int TS = M::O_V;                              // tables kept in shared memory (doubles)
  static constexpr size_t O_T = NB * size_t(BUF);
  // per-lane volume-point columns [lane n][2 points][psi(4) | w dpsi (a, i) (12)]; lane stride 34
  // doubles (272 B = 16 mod 128), so the four lanes' 16-byte reads fall in different banks (with
  // 32 they were 4-way conflicts: 22 % of the kernel's shared-memory wavefronts)
  static constexpr int VLS = 34;
  static constexpr size_t O_VL = O_T + size_t(TS) * 8;
  static constexpr size_t O_SC = O_VL + 4 * VLS * 8;              // [warp][8 elements][20] neighbour coefficients
  static constexpr size_t O_BAR = O_SC + size_t(CT / 32) * 8 * 20 * 8;
  static constexpr size_t SMEM = O_BAR + 32 + 80;                // full[NB] barriers, ghost states
  static_assert(SMEM <= 227 * 1024, "modal p = 1 tile buffers do not fit in shared memory");
};

template <int MODE>
__global__ void __launch_bounds__(ML4::NT, 1) modal_lo4_kernel(const StageArgs A) {
  using L = ML4;
  using M = MS<1>;
  constexpr int NP = 4, NQ = 8, NQF = 4, T = L::T, NT = L::NT, NB = L::NB;
  extern __shared__ __align__(128) unsigned char smem[];
  auto bufQ = [&](int b) { return reinterpret_cast<double*>(smem + size_t(b) * L::BUF); };
  auto bufR = [&](int b) { return reinterpret_cast<double*>(smem + size_t(b) * L::BUF + L::BQ); };
  auto bufG = [&](int b) { return reinterpret_cast<double*>(smem + size_t(b) * L::BUF + 2 * L::BQ); };
  auto bufN = [&](int b) { return reinterpret_cast<int*>(smem + size_t(b) * L::BUF + 2 * L::BQ + L::BG); };
  auto bufC = [&](int b) { return reinterpret_cast<uint8_t*>(smem + size_t(b) * L::BUF + 2 * L::BQ + L::BG + L::BN); };
  auto bufM = [&](int b) { return reinterpret_cast<uint8_t*>(smem + size_t(b) * L::BUF + 2 * L::BQ + L::BG + L::BN + L::BC); };
  double* sT = reinterpret_cast<double*>(smem + L::O_T);
  double* sVL = reinterpret_cast<double*>(smem + L::O_VL);
  double* sSC = reinterpret_cast<double*>(smem + L::O_SC);
  uint64_t* sBar = reinterpret_cast<uint64_t*>(smem + L::O_BAR);
  double* sGh = reinterpret_cast<double*>(sBar + 4);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if ((DG_PDL >> 1) & 1) pdl_launch_dependents();
  const double* Tg = A.op;
  for (int i = tid; i < L::TS; i += NT) sT[i] = Tg[i];
  // lane n's volume-point columns: point q = n + 4 h: psi_i(q), then (w dpsi_i/dxi_a)(q) at [a][i]
  if (tid < 4 * 32) {
    const int n = tid >> 5, r = tid & 31, h = r >> 4, k = r & 15, q = n + 4 * h;
    sVL[n * L::VLS + r] = k < 4 ? Tg[M::O_VQ + q * NP + k] : Tg[M::O_DQ + (((k - 4) >> 2) * NP + ((k - 4) & 3)) * NQ + q];
  }
  if (tid == 0)
    for (int b = 0; b < NB; ++b) mbar_init(&sBar[b], 1);
  if (tid == 32) {
    double qi[5];
    inflow_state(A, qi);
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      sGh[c] = A.qinf[c];
      sGh[5 + c] = qi[c];
    }
  }
  __syncthreads();
  if ((DG_PDL >> 1) & 1) pdl_wait();
  const int ntiles = (A.e_end - A.e_begin + T - 1) / T;
  const int nmine = (ntiles > (int)blockIdx.x) ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  auto tile_e0 = [&](int jj) { return A.e_begin + (int(blockIdx.x) + jj * int(gridDim.x)) * T; };
  auto tile_full = [&](int jj) { return A.e_end - tile_e0(jj) >= T; };
  constexpr int BAR_DONE = 1;

  if (warp == L::CT / 32) {
    // ======================= IO warp
    auto issue_load = [&](int jj) {
      const int b = jj % NB;
      if (tile_full(jj)) {
        const size_t e0 = size_t(tile_e0(jj));
        fence_proxy_async();
        mbar_arrive_expect_tx(&sBar[b], (MODE == MODE_UPDATE ? 2 * L::BQ : L::BQ) + L::BG + L::BN + L::BC + L::BM);
        tma_load_1d(bufQ(b), A.Qin + e0 * 5 * NP, L::BQ, &sBar[b]);
        if (MODE == MODE_UPDATE) tma_load_1d(bufR(b), A.res + e0 * 5 * NP, L::BQ, &sBar[b]);
        tma_load_1d(bufG(b), A.geo + e0 * GEO, L::BG, &sBar[b]);
        tma_load_1d(bufN(b), A.nbr + e0 * 4, L::BN, &sBar[b]);
        tma_load_1d(bufC(b), A.code + e0 * 4, L::BC, &sBar[b]);
        tma_load_1d(bufM(b), A.mtid + e0 * 8, L::BM, &sBar[b]);
      } else {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&sBar[b])) : "memory");
      }
    };
    if (lane == 0)
      for (int jj = 0; jj < NB && jj < nmine; ++jj) issue_load(jj);
    for (int j = 0; j < nmine; ++j) {
      const int b = j % NB;
      nbar_sync(BAR_DONE + b, NT);
      if (lane == 0) {
        const bool st = MODE == MODE_UPDATE && tile_full(j);
        if (st) {
          const size_t e0 = size_t(tile_e0(j));
          fence_proxy_async();
          tma_store_1d(A.Qout + e0 * 5 * NP, bufQ(b), L::BQ);
          tma_store_1d(A.res + e0 * 5 * NP, bufR(b), L::BQ);
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
        if (j + NB < nmine) {
          if (st) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
          issue_load(j + NB);
        }
      }
      __syncwarp();
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    return;
  }

  // ======================= compute warps: lane (es, n)
  const double gamma = A.gamma, gm1 = A.gamma - 1.0;
  const int es = tid >> 2, n = tid & 3;
  const double* vl = sVL + n * L::VLS;
  double* sc = sSC + (warp * 8 + (lane >> 2)) * 20;
  const double wfn = sT[M::O_WF + n];
  const bool o1 = n & 1, o2 = (n & 2) != 0;
  for (int j = 0; j < nmine; ++j) {
    const int b = j % NB;
    const int e0 = tile_e0(j);
    const int ne = min(T, A.e_end - e0);
    const bool full = ne == T;
    double* c_s = bufQ(b) + es * 5 * NP;
    double* r_s = bufR(b) + es * 5 * NP;
    double* g_s = bufG(b) + es * GEO;
    int* n_s = bufN(b) + es * 4;
    uint8_t* k_s = bufC(b) + es * 4;
    uint8_t* t_s = bufM(b) + es * 8;
    mbar_wait(&sBar[b], (j / NB) & 1);
    const bool active = es < ne;
    const size_t eg = size_t(e0) + (active ? es : ne - 1);
    if (!full) {
#pragma unroll
      for (int c = 0; c < 5; ++c) c_s[c * NP + n] = __ldg(A.Qin + eg * 5 * NP + c * NP + n);
      for (int i = n; i < GEO; i += 4) g_s[i] = __ldg(A.geo + eg * GEO + i);
      n_s[n] = __ldg(A.nbr + eg * 4 + n);
      k_s[n] = A.code[eg * 4 + n];
      t_s[2 * n] = A.mtid[eg * 8 + 2 * n];
      t_s[2 * n + 1] = A.mtid[eg * 8 + 2 * n + 1];
      __syncwarp();
    }
    // ---- mode n of the face neighbours' coefficients: face 0 now (behind the volume points),
    //      face f + 1 while face f is computed (one face of look-ahead keeps 10 registers busy,
    //      all four at once spilled)
    int tagf[4], nbf[4];
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const int code = k_s[f];
      tagf[f] = code >= CODE_BC ? code - CODE_BC : 0;
      nbf[f] = code < CODE_GHOST ? n_s[f] : -1;
    }
    double cn[5];
    auto gather = [&](int f) {
#pragma unroll
      for (int c = 0; c < 5; ++c) cn[c] = 0.0;
      if (nbf[f] >= 0) {
        const double* q2 = A.Qin + size_t(nbf[f]) * 5 * NP + n;
#pragma unroll
        for (int c = 0; c < 5; ++c) cn[c] = __ldg(q2 + c * NP);
      }
    };
    gather(0);
    // ---- volume points n and n + 4
    double part[5][NP];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const double2 v01 = *reinterpret_cast<const double2*>(vl + 16 * h);
      const double2 v23 = *reinterpret_cast<const double2*>(vl + 16 * h + 2);
      double u[5];
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        const double2 a01 = *reinterpret_cast<const double2*>(c_s + c * NP);
        const double2 a23 = *reinterpret_cast<const double2*>(c_s + c * NP + 2);
        u[c] = fma(v23.y, a23.y, fma(v23.x, a23.x, fma(v01.y, a01.y, v01.x * a01.x)));
      }
      const double ri = rcp_nr(u[0]);
      const double vx = u[1] * ri, vy = u[2] * ri, vz = u[3] * ri;
      const double p = gm1 * (u[4] - 0.5 * (u[1] * vx + u[2] * vy + u[3] * vz));
      if (active && !state_ok(u[0], p, u[1], u[2], u[3], u[4])) flag_blowup(A.flag, A.gid[eg]);
      const double pd = p - A.pref, Ep = u[4] + p;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double cx = g_s[3 * a], cy = g_s[3 * a + 1], cz = g_s[3 * a + 2];
        const double U = cx * vx + cy * vy + cz * vz;
        double fl[5];
        fl[0] = u[0] * U;
        fl[1] = fma(cx, pd, u[1] * U);
        fl[2] = fma(cy, pd, u[2] * U);
        fl[3] = fma(cz, pd, u[3] * U);
        fl[4] = Ep * U;
        const double2 d01 = *reinterpret_cast<const double2*>(vl + 16 * h + 4 + 4 * a);
        const double2 d23 = *reinterpret_cast<const double2*>(vl + 16 * h + 4 + 4 * a + 2);
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          const bool first = h == 0 && a == 0;
          part[c][0] = first ? d01.x * fl[c] : fma(d01.x, fl[c], part[c][0]);
          part[c][1] = first ? d01.y * fl[c] : fma(d01.y, fl[c], part[c][1]);
          part[c][2] = first ? d23.x * fl[c] : fma(d23.x, fl[c], part[c][2]);
          part[c][3] = first ? d23.y * fl[c] : fma(d23.y, fl[c], part[c][3]);
        }
      }
    }
    // ---- faces: point n of each face
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const double nx = g_s[9 + 4 * f], ny = g_s[9 + 4 * f + 1], nz = g_s[9 + 4 * f + 2];
      const double scw = g_s[9 + 4 * f + 3] * wfn;
      // the neighbour's 20 coefficients through the warp's scratch slot of this element
      __syncwarp();
#pragma unroll
      for (int c = 0; c < 5; ++c) sc[c * NP + n] = cn[c];
      __syncwarp();
      if (f < 3) gather(f + 1);
      const double* to = sT + M::O_PSTD + int(t_s[2 * f]) * NQF * NP + n * NP;
      const double* tn = sT + M::O_PSTD + int(t_s[2 * f + 1]) * NQF * NP + n * NP;
      const double2 o01 = *reinterpret_cast<const double2*>(to);
      const double2 o23 = *reinterpret_cast<const double2*>(to + 2);
      double um[5], up[5];
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        const double2 a01 = *reinterpret_cast<const double2*>(c_s + c * NP);
        const double2 a23 = *reinterpret_cast<const double2*>(c_s + c * NP + 2);
        um[c] = fma(o23.y, a23.y, fma(o23.x, a23.x, fma(o01.y, a01.y, o01.x * a01.x)));
      }
      if (tagf[f] == 0) {
        const double2 n01 = *reinterpret_cast<const double2*>(tn);
        const double2 n23 = *reinterpret_cast<const double2*>(tn + 2);
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          const double2 a01 = *reinterpret_cast<const double2*>(sc + c * NP);
          const double2 a23 = *reinterpret_cast<const double2*>(sc + c * NP + 2);
          up[c] = fma(n23.y, a23.y, fma(n23.x, a23.x, fma(n01.y, a01.y, n01.x * a01.x)));
        }
      } else if (tagf[f] == 1) {   // slip wall: mirror the normal momentum (Eq. 4)
        const double mn = um[1] * nx + um[2] * ny + um[3] * nz;
        up[0] = um[0];
        up[1] = um[1] - 2.0 * mn * nx;
        up[2] = um[2] - 2.0 * mn * ny;
        up[3] = um[3] - 2.0 * mn * nz;
        up[4] = um[4];
      } else {                     // pass-through (2) / inflow (3)
        const double* gh = sGh + (tagf[f] == 2 ? 0 : 5);
#pragma unroll
        for (int c = 0; c < 5; ++c) up[c] = gh[c];
      }
      const double rim = rcp_nr(um[0]);
      const double unm = (um[1] * nx + um[2] * ny + um[3] * nz) * rim;
      const double pm = gm1 * (um[4] - 0.5 * (um[1] * um[1] + um[2] * um[2] + um[3] * um[3]) * rim);
      const double rip = rcp_nr(up[0]);
      const double unp = (up[1] * nx + up[2] * ny + up[3] * nz) * rip;
      const double pp = gm1 * (up[4] - 0.5 * (up[1] * up[1] + up[2] * up[2] + up[3] * up[3]) * rip);
      double lam = fmax(fabs(unm) + sqrt_nr(gamma * pm * rim), fabs(unp) + sqrt_nr(gamma * pp * rip));
      if (A.lambda_mode == 0) {    // face max over the face's four points = the element's four lanes
        long long a = __double_as_longlong(lam);
        long long o = __shfl_xor_sync(0xffffffffu, a, 1);
        a = a > o ? a : o;
        o = __shfl_xor_sync(0xffffffffu, a, 2);
        lam = __longlong_as_double(a > o ? a : o);
      }
      // F*_n - (ambient shift) = (n.F(u-) + n.F(u+)) / 2 - lam (u+ - u-) / 2, weighted by Fscale w
      const double pdm = pm - A.pref, pdp = pp - A.pref;
      double fs[5];
      fs[0] = 0.5 * (um[0] * unm + up[0] * unp);
      fs[1] = 0.5 * (fma(pdm, nx, um[1] * unm) + fma(pdp, nx, up[1] * unp));
      fs[2] = 0.5 * (fma(pdm, ny, um[2] * unm) + fma(pdp, ny, up[2] * unp));
      fs[3] = 0.5 * (fma(pdm, nz, um[3] * unm) + fma(pdp, nz, up[3] * unp));
      fs[4] = 0.5 * ((um[4] + pm) * unm + (up[4] + pp) * unp);
      const double hl = 0.5 * lam;
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        const double w = -scw * fma(-hl, up[c] - um[c], fs[c]);
        part[c][0] = fma(o01.x, w, part[c][0]);
        part[c][1] = fma(o01.y, w, part[c][1]);
        part[c][2] = fma(o23.x, w, part[c][2]);
        part[c][3] = fma(o23.y, w, part[c][3]);
      }
    }
    // ---- sum the four lanes' partials; lane n keeps mode n
    double rhs[5];
    {
      double k0[5], k1[5];
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        const double s0 = __shfl_xor_sync(0xffffffffu, o1 ? part[c][0] : part[c][1], 1);
        const double s1 = __shfl_xor_sync(0xffffffffu, o1 ? part[c][2] : part[c][3], 1);
        k0[c] = (o1 ? part[c][1] : part[c][0]) + s0;
        k1[c] = (o1 ? part[c][3] : part[c][2]) + s1;
      }
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        const double s = __shfl_xor_sync(0xffffffffu, o2 ? k0[c] : k1[c], 2);
        rhs[c] = (o2 ? k1[c] : k0[c]) + s;
      }
    }
    if (MODE == MODE_UPDATE) {
      if (full) {
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          const double rr = fma(A.a, r_s[c * NP + n], A.dt * rhs[c]);
          const double qo = c_s[c * NP + n];
          r_s[c * NP + n] = rr;
          c_s[c * NP + n] = fma(A.b, rr, qo);
        }
      } else if (active) {
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          const size_t gi = eg * 5 * NP + c * NP + n;
          const double rr = fma(A.a, __ldg(A.res + gi), A.dt * rhs[c]);
          A.res[gi] = rr;
          A.Qout[gi] = fma(A.b, rr, c_s[c * NP + n]);
        }
      }
    } else {
      // rhs out as nodal values V dc/dt (the ABI state is nodal): node n needs the four modes
      const int l0 = lane & ~3;
      const size_t pe = size_t(A.pub[eg]);
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < NP; ++i) acc = fma(__ldg(Tg + M::O_V + n * NP + i), __shfl_sync(0xffffffffu, rhs[c], l0 + i), acc);
        if (active) A.out[(size_t(c) * A.Kpub + pe) * NP + n] = acc;
      }
    }
    if (MODE == MODE_UPDATE && full) fence_proxy_async();
    nbar_arrive(BAR_DONE + b, NT);
  }
}

}  // namespace dgk
