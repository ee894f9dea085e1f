// Tile kernel of the paper's modal-quadrature scheme (Appendix A,
// P:396-419; reading A23).  Same arithmetic as modal_warp_kernel (kernels.cuh), laid
// out for throughput: a persistent CTA (512 threads) walks tiles of EB elements; the next tile's
// coefficients, geometry and connectivity arrive by TMA while the current one is processed, the
// neighbours' coefficients by cp.async, and every phase runs over the whole tile with all
// threads:
//   V  values of the tile's polynomials at the (p+1)^3 volume points, contravariant fluxes there
//      (item = element x point);
//   F  both traces at the owner's (p+1)^2 points of every face (item = element x face x point):
//      own = T_own c, neighbour = T_nb c_nb with per-face tables (host-chosen ids: the standard
//      points of the owner or the owner's points carried onto this face), ghosts at boundaries,
//      wave speeds; after a barrier the face max and the LLF flux weighted by Fscale w;
//   P  projection onto the basis, dc_i/dt = sum_q,a (w dpsi_i/dxi_a)(q) Ft_a(q)
//                                         - sum_f,q psi_i(q_f) [Fscale w F*_n](q_f),
//      as four interleaved partial sums (item = element x field x mode), and the LSERK update
//      with coalesced global loads and stores ([K][5][Np] order = item order).
// Tables live in shared memory (for p = 3 the 96 carried-point tables stay in global memory).
#pragma once
#include "kernels.cuh"

namespace dgk {

#ifndef DG_MI    // interpolation to the volume points on DMMA (1) or DFMA dot products (0)
#define DG_MI 1
#endif
// face projection: 2 = DMMA per (element, mode tile), 1 = item (row, face), 0 = item (row, mode);
// default 2 at p = 3 (7.9 -> 9.3 GDOF/s), 0 at p <= 2 (p = 2: 12.8 vs 11.8)
#ifdef DG_MFP
#define DG_MFP_P(P) DG_MFP
#else
#define DG_MFP_P(P) ((P) >= 3 ? 2 : 0)
#endif

template <int P>
struct MT {
  using M = MS<P>;
  static constexpr int NP = M::NP, NQ = M::NQ, NQF = M::NQF;
  static constexpr int EB = P == 1 ? 32 : P == 2 ? 16 : 8;
  static constexpr int NT = 512;
  static constexpr int ROWS = 5 * EB;
  static constexpr bool PMAP_SMEM = P <= 2;
  // table prefix kept in shared memory: WQ, VQ, DQ, WF, PSTD (+ PMAP for p <= 2)
  static constexpr int TS = PMAP_SMEM ? M::O_V : M::O_PMAP;
  // volume projection on the FP64 tensor cores (DMMA m8n8k4): rows (element, field), k = a NQ + q
  // (padded to KVP), n = mode (padded to NPAD); FV rows strided == 4 or 12 (mod 16) doubles so
  // the A fragments are conflict-free
  static constexpr int KV = 3 * NQ, KVP = (KV + 3) / 4 * 4, KS = KVP / 4;
  static constexpr int NPAD = (NP + 7) / 8 * 8, NTL = NPAD / 8;
  static constexpr int fvs() {
    int x = KVP;
    while (x % 16 != 4 && x % 16 != 12) ++x;
    return x;
  }
  static constexpr int FVS = fvs();     // FV row (element, field): columns a NQ + q
  static constexpr int MT8 = ROWS / 8, UNITS = MT8 * NTL;
  // the k range of each unit is split KP ways so every warp gets work; the KP partial results go
  // to separate buffers (in the neighbours' coefficient region, dead by then) and are summed in a
  // fixed order -- deterministic
  // (k-split 2-4 ways so every warp gets a unit measured slower, p = 1 / 2 / 3: 16.9 / 12.3 / 9.5
  // vs 19.2 / 13.5 / 9.7 GDOF/s)
  static constexpr int KP = 1;
  // interpolation to the volume points on DMMA: A = the tile's coefficients as loaded ([row][NP];
  // k past NP meets zero B rows -- the values read there are the next row's coefficients or the
  // geometry behind the block, finite), n = point (NQ padded to NTQ tiles), result into the FS
  // buffer (free until the face phase) with row stride FSS >= NQ
  static constexpr int KI = (NP + 3) / 4 * 4, KSI = KI / 4, NTQ = (NQ + 7) / 8, UNITS_I = MT8 * NTQ;
  static_assert(ROWS % 8 == 0, "DMMA row tiles");
  static constexpr int FSS = 4 * NQF;   // FS row: columns f NQF + q
  // input buffer (TMA): coefficients, geometry, neighbours, codes, face table ids
  static constexpr uint32_t BC_ = uint32_t(EB) * 5 * NP * 8;
  static constexpr uint32_t BG = uint32_t(EB) * GEO * 8;
  static constexpr uint32_t BN = uint32_t(EB) * 16;
  static constexpr uint32_t BK = uint32_t(EB) * 4;
  static constexpr uint32_t BT = uint32_t(EB) * 8;
  static constexpr uint32_t BIN = BC_ + BG + BN + BK + BT;
  static_assert(BC_ % 16 == 0 && BG % 16 == 0 && BN % 16 == 0 && BK % 16 == 0 && BT % 16 == 0, "TMA sizes");
  // shared-memory layout (bytes)
  static constexpr size_t O_T = 0;
  static constexpr size_t O_IN = (size_t(TS) * 8 + 127) / 128 * 128;
  static constexpr size_t O_CN = O_IN + 2 * size_t(BIN);
  static constexpr size_t O_FV = O_CN + size_t(EB) * 20 * NP * 8;
  static constexpr size_t O_FS = O_FV + size_t(ROWS) * FVS * 8;
  static constexpr size_t O_LAM = O_FS + size_t(ROWS) * FSS * 8;
  static constexpr size_t O_FR = O_LAM + size_t(EB) * 4 * NQF * 8;       // B fragments of the volume projection
  static constexpr size_t O_FI = O_FR + size_t(KS) * NTL * 32 * 8;         // B fragments of the interpolation
  static constexpr size_t O_RV = O_CN;   // volume-projection result [ROWS][NP] (the neighbours' coefficients are dead by then)
  static_assert(size_t(KP) * ROWS * NP <= size_t(EB) * 20 * NP && 4 * NQF >= NQ, "buffer aliases");
  static constexpr size_t O_BAR = O_FI + size_t(KSI) * NTQ * 32 * 8;
  static constexpr size_t SMEM = O_BAR + 16;
  static_assert(SMEM <= 227 * 1024, "modal tile does not fit in shared memory");
  static constexpr int FR = (EB * 4 * NQF + NT - 1) / NT;   // face rounds
  static constexpr int PR = (ROWS * NP + NT - 1) / NT;      // projection rounds
};

__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

template <int P, int MODE>
__global__ void __launch_bounds__(MT<P>::NT, 1) modal_tile_kernel(const StageArgs A) {
  using M = MS<P>;
  using W = MT<P>;
  constexpr int NP = W::NP, NQ = W::NQ, NQF = W::NQF, EB = W::EB, NT = W::NT;
  extern __shared__ __align__(128) unsigned char smem[];
  double* sT = reinterpret_cast<double*>(smem + W::O_T);
  unsigned char* in0 = smem + W::O_IN;
  double* sCN = reinterpret_cast<double*>(smem + W::O_CN);
  double* sFV = reinterpret_cast<double*>(smem + W::O_FV);
  double* sFS = reinterpret_cast<double*>(smem + W::O_FS);
  double* sLAM = reinterpret_cast<double*>(smem + W::O_LAM);
  double* sFR = reinterpret_cast<double*>(smem + W::O_FR);
  double* sRV = reinterpret_cast<double*>(smem + W::O_RV);
  uint64_t* sBar = reinterpret_cast<uint64_t*>(smem + W::O_BAR);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const double* T = A.op;
  const double gamma = A.gamma, gm1 = A.gamma - 1.0;

  for (int i = tid; i < W::TS; i += NT) sT[i] = T[i];
  // B fragments of (w dpsi_i/dxi_a)(q): lane holds B[k = 4 ks + t][n = 8 nt + g] = DQ(a, n, q), k = a NQ + q
  for (int idx = tid; idx < W::KS * W::NTL * 32; idx += NT) {
    const int ks = idx / (W::NTL * 32), r = idx - ks * W::NTL * 32, nt = r >> 5, ln = r & 31;
    const int k = 4 * ks + (ln & 3), n = nt * 8 + (ln >> 2);
    const int a = k / NQ, q = k - a * NQ;
    sFR[idx] = (k < W::KV && n < NP) ? T[M::O_DQ + (a * NP + n) * NQ + q] : 0.0;
  }
  for (int i = tid; i < W::ROWS * W::FVS; i += NT) sFV[i] = 0.0;   // padding columns stay 0
  double* sFI = reinterpret_cast<double*>(smem + W::O_FI);
  // B fragments of psi_i(q): lane holds B[k = 4 ks + t][n = 8 nt + g] = VQ(q = n, i = k)
  for (int idx = tid; idx < W::KSI * W::NTQ * 32; idx += NT) {
    const int ks = idx / (W::NTQ * 32), r = idx - ks * W::NTQ * 32, nt = r >> 5, ln = r & 31;
    const int k = 4 * ks + (ln & 3), n = nt * 8 + (ln >> 2);
    sFI[idx] = (k < NP && n < NQ) ? T[M::O_VQ + n * NP + k] : 0.0;
  }
  if (tid == 0) {
    mbar_init(&sBar[0], 1);
    mbar_init(&sBar[1], 1);
  }
  __syncthreads();
  auto ftab = [&](int t) -> const double* {   // face table t: 0-3 standard points, 4+ carried points
    if (W::PMAP_SMEM || t < 4) return sT + M::O_PSTD + t * NQF * NP;
    return T + M::O_PSTD + t * NQF * NP;
  };
  auto bufC = [&](int b) { return reinterpret_cast<double*>(in0 + b * W::BIN); };
  auto bufG = [&](int b) { return reinterpret_cast<double*>(in0 + b * W::BIN + W::BC_); };
  auto bufN = [&](int b) { return reinterpret_cast<int*>(in0 + b * W::BIN + W::BC_ + W::BG); };
  auto bufK = [&](int b) { return in0 + b * W::BIN + W::BC_ + W::BG + W::BN; };
  auto bufT = [&](int b) { return in0 + b * W::BIN + W::BC_ + W::BG + W::BN + W::BK; };

  const int ntiles = (A.e_end - A.e_begin + EB - 1) / EB;
  const int nmine = (ntiles > (int)blockIdx.x) ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  auto tile_e0 = [&](int jj) { return A.e_begin + (int(blockIdx.x) + jj * int(gridDim.x)) * EB; };
  // full tiles by TMA (thread 0); the partial last tile by plain loads of all threads, zero-filled
  auto fetch = [&](int jj) {
    const int e0 = tile_e0(jj);
    const int b = jj & 1;
    if (A.e_end - e0 >= EB) {
      if (tid == 0) {
        fence_proxy_async();
        mbar_arrive_expect_tx(&sBar[b], W::BIN);
        tma_load_1d(bufC(b), A.Qin + size_t(e0) * 5 * NP, W::BC_, &sBar[b]);
        tma_load_1d(bufG(b), A.geo + size_t(e0) * GEO, W::BG, &sBar[b]);
        tma_load_1d(bufN(b), A.nbr + size_t(e0) * 4, W::BN, &sBar[b]);
        tma_load_1d(bufK(b), A.code + size_t(e0) * 4, W::BK, &sBar[b]);
        tma_load_1d(bufT(b), A.mtid + size_t(e0) * 8, W::BT, &sBar[b]);
      }
    } else {
      const int ne = A.e_end - e0;
      for (int i = tid; i < EB * 5 * NP; i += NT) bufC(b)[i] = i < ne * 5 * NP ? A.Qin[size_t(e0) * 5 * NP + i] : 0.0;
      for (int i = tid; i < EB * GEO; i += NT) bufG(b)[i] = i < ne * GEO ? A.geo[size_t(e0) * GEO + i] : 0.0;
      for (int i = tid; i < EB * 4; i += NT) {
        bufN(b)[i] = i < ne * 4 ? A.nbr[size_t(e0) * 4 + i] : 0;
        bufK(b)[i] = i < ne * 4 ? A.code[size_t(e0) * 4 + i] : uint8_t(CODE_BC + 2);
      }
      for (int i = tid; i < EB * 8; i += NT) bufT(b)[i] = i < ne * 8 ? A.mtid[size_t(e0) * 8 + i] : uint8_t(0);
    }
  };
  if (nmine > 0) fetch(0);
  __syncthreads();   // a partial tile 0 stored by plain loads

  for (int j = 0; j < nmine; ++j) {
    const int e0 = tile_e0(j);
    const int ne = min(EB, A.e_end - e0);
    const int b = j & 1;
    // the other buffer (tile j-1) was released by the barrier that ended tile j-1
    if (j + 1 < nmine) {
      if (A.e_end - tile_e0(j + 1) >= EB) fetch(j + 1);
    }
    if (ne == EB) mbar_wait(&sBar[b], (j >> 1) & 1);
    const double* cS = bufC(b);
    const double* gS = bufG(b);
    const int* nS = bufN(b);
    const uint8_t* kS = bufK(b);
    const uint8_t* tS = bufT(b);

    // ---- neighbours' coefficients (16-byte cp.async -- a face's block is 5 Np doubles, a multiple
    //      of 2 -- waited for before the face phase)
    for (int i2 = tid; i2 < EB * 10 * NP; i2 += NT) {
      const int i = 2 * i2;
      const int e = i / (20 * NP), r1 = i - e * 20 * NP, f = r1 / (5 * NP), r0 = r1 - f * 5 * NP;
      const int code = kS[e * 4 + f];
      if (e < ne && code < CODE_GHOST) cp_async16(sCN + i, A.Qin + size_t(nS[e * 4 + f]) * 5 * NP + r0);
    }

    // ---- V: values at the volume points (DMMA into the FS buffer), then the contravariant fluxes
    for (int u0 = warp; DG_MI && u0 < W::UNITS_I; u0 += NT / 32) {
      const int rt = u0 / W::NTQ, nt = u0 - rt * W::NTQ;
      double acc[2] = {0.0, 0.0};
      const double* X = cS + (rt * 8 + g) * NP + t4;
      const double* B = sFI + nt * 32 + lane;
#pragma unroll
      for (int ks = 0; ks < W::KSI; ++ks) dmma_8x8x4(acc, X[4 * ks], B[ks * W::NTQ * 32]);
      const int n0 = nt * 8 + 2 * t4;
      double* o = sFS + (rt * 8 + g) * W::FSS;
      if (n0 < NQ) o[n0] = acc[0];
      if (n0 + 1 < NQ) o[n0 + 1] = acc[1];
    }
    __syncthreads();
    for (int v = tid; v < EB * NQ; v += NT) {
      const int e = v / NQ, q = v - e * NQ;
      double u[5];
      if (DG_MI) {
#pragma unroll
        for (int c = 0; c < 5; ++c) u[c] = sFS[(e * 5 + c) * W::FSS + q];
      } else {
        const double* c_s = cS + e * 5 * NP;
        const double* vq = sT + M::O_VQ + q * NP;
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          double acc = 0.0;
#pragma unroll
          for (int i = 0; i < NP; ++i) acc = fma(vq[i], c_s[c * NP + i], acc);
          u[c] = acc;
        }
      }
      const bool act = e < ne;
      if (!act) u[0] = 1.0, u[4] = 2.5;   // padding elements: a harmless state
      const double ri = 1.0 / u[0];
      const double vx = u[1] * ri, vy = u[2] * ri, vz = u[3] * ri;
      const double p = gm1 * (u[4] - 0.5 * (u[1] * vx + u[2] * vy + u[3] * vz));
      if (act && !state_ok(u[0], p, u[1], u[2], u[3], u[4])) flag_blowup(A.flag, A.gid[e0 + e]);
      const double pd = p - A.pref, Ep = u[4] + p;
      const double* G = gS + e * GEO;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double cx = G[3 * a], cy = G[3 * a + 1], cz = G[3 * a + 2];
        const double U = cx * vx + cy * vy + cz * vz;
        double* o = sFV + (e * 5) * W::FVS + a * NQ + q;
        o[0] = u[0] * U;
        o[W::FVS] = fma(cx, pd, u[1] * U);
        o[2 * W::FVS] = fma(cy, pd, u[2] * U);
        o[3 * W::FVS] = fma(cz, pd, u[3] * U);
        o[4 * W::FVS] = Ep * U;
      }
    }
    cp_async_wait_all();
    __syncthreads();

    // ---- F: both traces at the face points, wave speeds
    double um[W::FR][5], up[W::FR][5];
#pragma unroll
    for (int rr = 0; rr < W::FR; ++rr) {
      const int v = tid + rr * NT;
      if (v >= EB * 4 * NQF) break;
      const int e = v / (4 * NQF), fq = v - e * 4 * NQF, f = fq / NQF, q = fq - f * NQF;
      const int code = kS[e * 4 + f];
      const double* Gf = gS + e * GEO + 9 + 4 * f;
      const double* to = ftab(tS[e * 8 + 2 * f]) + q * NP;
      const double* c_s = cS + e * 5 * NP;
      // 16-byte loads (Np is even, rows 16-byte aligned): half the shared-memory instructions of
      // the dot products, which bound this phase (DG_MDV2, p = 2: 13.0 -> see DESIGN.md)
      static_assert(NP % 2 == 0, "two modes per 16-byte load");
      double2 tov[NP / 2];
#pragma unroll
      for (int i = 0; i < NP / 2; ++i) tov[i] = reinterpret_cast<const double2*>(to)[i];
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int i = 0; i < NP / 2; ++i) {
          const double2 cv = reinterpret_cast<const double2*>(c_s + c * NP)[i];
          a0 = fma(tov[i].x, cv.x, a0);
          a1 = fma(tov[i].y, cv.y, a1);
        }
        um[rr][c] = a0 + a1;
      }
      if (e >= ne) um[rr][0] = 1.0, um[rr][4] = 2.5;
      if (code < CODE_GHOST && e < ne) {
        const double* tn = ftab(tS[e * 8 + 2 * f + 1]) + q * NP;
        const double* cn = sCN + (e * 4 + f) * 5 * NP;
        double2 tnv[NP / 2];
#pragma unroll
        for (int i = 0; i < NP / 2; ++i) tnv[i] = reinterpret_cast<const double2*>(tn)[i];
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          double a0 = 0.0, a1 = 0.0;
#pragma unroll
          for (int i = 0; i < NP / 2; ++i) {
            const double2 cv = reinterpret_cast<const double2*>(cn + c * NP)[i];
            a0 = fma(tnv[i].x, cv.x, a0);
            a1 = fma(tnv[i].y, cv.y, a1);
          }
          up[rr][c] = a0 + a1;
        }
      } else if (e < ne) {
        ghost_trace(A, code - CODE_BC, um[rr], Gf[0], Gf[1], Gf[2], up[rr]);
      } else {
#pragma unroll
        for (int c = 0; c < 5; ++c) up[rr][c] = um[rr][c];
      }
      auto speed = [&](const double (&w)[5]) {
        const double ri = 1.0 / w[0];
        const double un = (w[1] * Gf[0] + w[2] * Gf[1] + w[3] * Gf[2]) * ri;
        const double p = gm1 * (w[4] - 0.5 * (w[1] * w[1] + w[2] * w[2] + w[3] * w[3]) * ri);
        return fabs(un) + sqrt(gamma * p * ri);
      };
      sLAM[v] = fmax(speed(um[rr]), speed(up[rr]));
    }
    __syncthreads();
#pragma unroll
    for (int rr = 0; rr < W::FR; ++rr) {
      const int v = tid + rr * NT;
      if (v >= EB * 4 * NQF) break;
      const int e = v / (4 * NQF), fq = v - e * 4 * NQF, f = fq / NQF, q = fq - f * NQF;
      const double* Gf = gS + e * GEO + 9 + 4 * f;
      const double nx = Gf[0], ny = Gf[1], nz = Gf[2];
      double lam = sLAM[v];
      if (A.lambda_mode == 0) {
#pragma unroll
        for (int qq = 0; qq < NQF; ++qq) lam = fmax(lam, sLAM[e * 4 * NQF + f * NQF + qq]);
      }
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
      const double sc = e < ne ? Gf[3] * sT[M::O_WF + q] : 0.0;
      double* fs = sFS + (e * 5) * W::FSS + fq;
#pragma unroll
      for (int c = 0; c < 5; ++c) fs[c * W::FSS] = sc * (0.5 * (fm[c] + fp[c]) - 0.5 * lam * (up[rr][c] - um[rr][c]));
    }
    __syncthreads();

    // ---- P1: volume projection on DMMA, (row tile, n tile) units over the warps
    for (int u = warp; u < W::UNITS * W::KP; u += NT / 32) {
      const int kp = u % W::KP, u1 = u / W::KP, rt = u1 / W::NTL, nt = u1 - rt * W::NTL;
      const int ks0 = kp * W::KS / W::KP, ks1 = (kp + 1) * W::KS / W::KP;
      double acc[2] = {0.0, 0.0};
      const double* X = sFV + (rt * 8 + g) * W::FVS + t4;
      const double* B = sFR + nt * 32 + lane;
#pragma unroll 4
      for (int ks = ks0; ks < ks1; ++ks) dmma_8x8x4(acc, X[4 * ks], B[ks * W::NTL * 32]);
      const int n0 = nt * 8 + 2 * t4;
      double* o = sRV + size_t(kp) * W::ROWS * NP + (rt * 8 + g) * NP;
      if (n0 < NP) o[n0] = acc[0];
      if (n0 + 1 < NP) o[n0 + 1] = acc[1];
    }
    __syncthreads();
    // ---- P2: face projection, item = (row, face) computing every mode (one fs load feeds NP
    //      FMAs), summed over the 4 faces of the row (consecutive lanes) by two shuffles, added to
    //      the volume part
    // DG_MFP == 2: unit = (element, mode tile); A = the element's 5 FS rows (rows 5-7 zero),
    // B[k = f NQF + q][n = i] = psi_i at the face's points (the element's own face tables)
    for (int u = warp; DG_MFP_P(P) == 2 && u < EB * W::NTL; u += NT / 32) {
      const int e = u / W::NTL, nt = u - e * W::NTL;
      const double* fsr = sFS + (e * 5 + (g < 5 ? g : 0)) * W::FSS;
      const double* tb[4];
#pragma unroll
      for (int f = 0; f < 4; ++f) tb[f] = ftab(tS[e * 8 + 2 * f]);
      const int n = nt * 8 + g;
      double acc[2] = {0.0, 0.0};
#pragma unroll
      for (int ks = 0; ks < NQF; ++ks) {
        const int k = 4 * ks + t4, f = k / NQF, q = k - f * NQF;
        const double a0 = g < 5 ? fsr[k] : 0.0;
        const double b0 = n < NP ? tb[f][q * NP + n] : 0.0;
        dmma_8x8x4(acc, a0, b0);
      }
      const int n0 = nt * 8 + 2 * t4;
      if (g < 5) {
        double* o = sRV + (e * 5 + g) * NP;
        if (n0 < NP) o[n0] -= acc[0];
        if (n0 + 1 < NP) o[n0 + 1] -= acc[1];
      }
    }
    for (int v0 = 0; DG_MFP_P(P) == 1 && v0 < W::ROWS * 4; v0 += NT) {
      const int v = v0 + tid;
      const bool ok = v < W::ROWS * 4;
      const int row = ok ? v >> 2 : 0, f = v & 3, e = row / 5;
      const double* fs = sFS + row * W::FSS + f * NQF;
      const double* Pt = ftab(tS[e * 8 + 2 * f]);
      double part[NP];
#pragma unroll
      for (int i = 0; i < NP; ++i) part[i] = 0.0;
#pragma unroll
      for (int q = 0; q < NQF; ++q) {
        const double w = fs[q];
#pragma unroll
        for (int i = 0; i < NP; ++i) part[i] = fma(Pt[q * NP + i], w, part[i]);
      }
#pragma unroll
      for (int i = 0; i < NP; ++i) {
        part[i] += __shfl_xor_sync(0xffffffffu, part[i], 1);
        part[i] += __shfl_xor_sync(0xffffffffu, part[i], 2);
      }
      if (ok && f == 0) {
#pragma unroll
        for (int i = 0; i < NP; ++i) sRV[row * NP + i] -= part[i];
      }
    }
    __syncthreads();
    // ---- P3: the update (or rhs out); a thread takes two adjacent modes of a row (16-byte loads
    //      of the face tables, the residual and the state; one round at every order)
    constexpr int PR2 = (W::ROWS * NP / 2 + NT - 1) / NT;
    double2 rhs[PR2];
#pragma unroll
    for (int rr = 0; rr < PR2; ++rr) {
      const int v = 2 * (tid + rr * NT);
      rhs[rr] = make_double2(0.0, 0.0);
      if (v >= W::ROWS * NP) break;
      const int e = v / (5 * NP);
      double2 acc = *reinterpret_cast<const double2*>(sRV + v);
#pragma unroll
      for (int kp = 1; kp < W::KP; ++kp) {
        const double2 t2 = *reinterpret_cast<const double2*>(sRV + kp * W::ROWS * NP + v);
        acc.x += t2.x;
        acc.y += t2.y;
      }
      if (DG_MFP_P(P) == 0) {
        const int row = v / NP, i = v - row * NP;
        const double* fs = sFS + row * W::FSS;
        double ax[4] = {acc.x, 0.0, 0.0, 0.0}, ay[4] = {acc.y, 0.0, 0.0, 0.0};
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          const double* Pt = ftab(tS[e * 8 + 2 * f]) + i;
#pragma unroll
          for (int q = 0; q < NQF; ++q) {
            const double2 pt = *reinterpret_cast<const double2*>(Pt + q * NP);
            const double w = fs[f * NQF + q];
            ax[(f * NQF + q) & 3] = fma(-pt.x, w, ax[(f * NQF + q) & 3]);
            ay[(f * NQF + q) & 3] = fma(-pt.y, w, ay[(f * NQF + q) & 3]);
          }
        }
        acc.x = (ax[0] + ax[1]) + (ax[2] + ax[3]);
        acc.y = (ay[0] + ay[1]) + (ay[2] + ay[3]);
      }
      rhs[rr] = acc;
      if (MODE == MODE_UPDATE && e < ne) {
        const size_t gi = size_t(e0) * 5 * NP + v;
        const double2 r0 = *reinterpret_cast<const double2*>(A.res + gi);
        const double2 c0 = *reinterpret_cast<const double2*>(cS + v);
        double2 r2, q2;
        r2.x = fma(A.a, r0.x, A.dt * acc.x);
        r2.y = fma(A.a, r0.y, A.dt * acc.y);
        q2.x = fma(A.b, r2.x, c0.x);
        q2.y = fma(A.b, r2.y, c0.y);
        *reinterpret_cast<double2*>(A.res + gi) = r2;
        *reinterpret_cast<double2*>(A.Qout + gi) = q2;
      }
    }
    if (MODE == MODE_RHS) {   // V (dc/dt) into the public layout, staged in the FV region
      __syncthreads();
#pragma unroll
      for (int rr = 0; rr < PR2; ++rr) {
        const int v = 2 * (tid + rr * NT);
        if (v < W::ROWS * NP) *reinterpret_cast<double2*>(sFV + v) = rhs[rr];
      }
      __syncthreads();
      for (int v = tid; v < ne * 5 * NP; v += NT) {
        const int e = v / (5 * NP), cn = v - e * 5 * NP, c = cn / NP, n = cn - c * NP;
        const double* r_s = sFV + e * 5 * NP + c * NP;
        double acc = 0.0;
        for (int i = 0; i < NP; ++i) acc = fma(__ldg(T + M::O_V + n * NP + i), r_s[i], acc);
        A.out[(size_t(c) * A.Kpub + A.pub[e0 + e]) * NP + n] = acc;
      }
    }
    __syncthreads();   // the tile's buffers may be refilled / overwritten by tile j+1 (and j+2)
    if (j + 1 < nmine && A.e_end - tile_e0(j + 1) < EB) {
      fetch(j + 1);    // the partial last tile, by plain loads
      __syncthreads();
    }
  }
}

}  // namespace dgk
