// C-ABI entry points of libdg_b200 (include/dg.h): workspace binding, state
// I/O, RHS and RK stepping on sm_100a, NCCL face-trace halo exchange.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>

#include "ctx.h"
#include "kernels.cuh"
#include "spectrum.cuh"
#include "modal.cuh"
#include "lo.cuh"

namespace {

thread_local std::string g_err;

dg_status set_err(dg_ctx* c, dg_status st, const std::string& m) {
  if (c) c->err = m;
  g_err = m;
  return st;
}

#define CUDA_TRY(c, x)                                                                       \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess)                                                                   \
      return set_err(c, DG_ECUDA, std::string("CUDA: ") + cudaGetErrorString(e_) + " at " #x); \
  } while (0)

#define NCCL_TRY(c, x)                                                                    \
  do {                                                                                    \
    ncclResult_t r_ = (x);                                                                \
    if (r_ != ncclSuccess) return set_err(c, DG_ENCCL, std::string("NCCL: ") + ncclGetErrorString(r_)); \
  } while (0)

// Carpenter & Kennedy (1994) five-stage fourth-order 2N-storage RK (BASELINE.json configs)
const double LSERK_A[5] = {0.0, -567301805773.0 / 1357537059087.0, -2404267990393.0 / 2016746695238.0,
                           -3550918686646.0 / 2091501179385.0, -1275806237668.0 / 842570457699.0};
const double LSERK_B[5] = {1432997174477.0 / 9575080441755.0, 5161836677717.0 / 13612068292357.0,
                           1720146321549.0 / 2090206949498.0, 3134564353537.0 / 4481467310338.0,
                           2277821191437.0 / 14882151754819.0};
const double LSERK_C[5] = {0.0, 1432997174477.0 / 9575080441755.0, 2526269341429.0 / 6820363962896.0,
                           2006345519317.0 / 3224310063776.0, 2802321613138.0 / 2924317926251.0};
// Heun = the paper's RK2 in the same 2N-storage form
const double HEUN_A[2] = {0.0, -1.0};
const double HEUN_B[2] = {1.0, 0.5};
const double HEUN_C[2] = {0.0, 1.0};

int nstages(const dg_ctx* c) { return c->rk_scheme == DG_RK_HEUN ? 2 : 5; }
void coeffs(const dg_ctx* c, int s, double& a, double& b, double& cc) {
  if (c->rk_scheme == DG_RK_HEUN) {
    a = HEUN_A[s]; b = HEUN_B[s]; cc = HEUN_C[s];
  } else {
    a = LSERK_A[s]; b = LSERK_B[s]; cc = LSERK_C[s];
  }
}

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

// per-device SM count and kernel-attribute state (a process may drive contexts on several GPUs)
constexpr int MAXDEV = 64;
int g_num_sms[MAXDEV] = {0};
int cur_dev() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev >= 0 && dev < MAXDEV ? dev : 0;
}
int num_sms() {
  const int dev = cur_dev();
  if (!g_num_sms[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    g_num_sms[dev] = n > 0 ? n : 148;
  }
  return g_num_sms[dev];
}
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: remember it per kernel and device
template <typename F>
cudaError_t ensure_smem_attr(F* kern, size_t smem, uint64_t& done_mask) {
  const int dev = cur_dev();
  if (done_mask >> dev & 1) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e == cudaSuccess) done_mask |= uint64_t(1) << dev;
  return e;
}
// persistent stage grid: one CTA per SM, capped by the ctx's max_ctas (dg_set_max_ctas)
int stage_grid(int ntiles, int max_ctas) {
  int g = std::min(ntiles, num_sms());
  if (max_ctas > 0) g = std::min(g, max_ctas);
  return g;
}

// ---------------------------------------------------------------- kernel dispatch
// stage launch, optionally with programmatic stream serialization (kernels.cuh DG_PDL)
template <typename... KArgs, typename... Args>
cudaError_t launch_stage_kernel(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t st, bool pdl,
                                Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <int N, int MODE>
cudaError_t launch_ho_n(const dgk::StageArgs& A, int max_ctas, cudaStream_t st) {
  using H = dgk::HO<N>;
  static uint64_t attr = 0;
  cudaError_t e = ensure_smem_attr(dgk::stage_ho_kernel<N, MODE>, H::SMEM, attr);
  if (e != cudaSuccess) return e;
  const int ntiles = (A.e_end - A.e_begin + H::EB - 1) / H::EB;
  if (ntiles <= 0) return cudaSuccess;
  dgk::stage_ho_kernel<N, MODE><<<stage_grid(ntiles, max_ctas), H::NT, H::SMEM, st>>>(A);
  return cudaGetLastError();
}

template <int N, int MODE, int V = 0>
cudaError_t launch_ws_n(const dgk::StageArgs& A, int max_ctas, cudaStream_t st) {
  using W = dgk::WS<N, V>;
  const int ntiles = (A.e_end - A.e_begin + W::EB - 1) / W::EB;
  if (ntiles <= 0) return cudaSuccess;
  if constexpr (N == 2 && V == 0) {
    // small meshes: the 48-element tile would leave SMs without a tile -- the 32-element variant
    if (ntiles < num_sms()) return launch_ws_n<N, MODE, 1>(A, max_ctas, st);
  }
  static uint64_t attr = 0;
  cudaError_t e = ensure_smem_attr(dgk::stage_ws_kernel<N, MODE, V>, W::SMEM, attr);
  if (e != cudaSuccess) return e;
  return launch_stage_kernel(dgk::stage_ws_kernel<N, MODE, V>, stage_grid(ntiles, max_ctas), W::NT, W::SMEM, st,
                             (DG_PDL >> N) & 1, A);
}

// N = 1, four lanes per element (lo.cuh stage_lo4_kernel); DG_LO4 = 0 keeps the DMMA kernel
#ifndef DG_LO4
#define DG_LO4 1
#endif
template <int MODE>
cudaError_t launch_lo4(const dg_ctx* c, const dgk::StageArgs& A, int max_ctas, cudaStream_t st) {
  using L = dgk::LO4;
  static uint64_t attr = 0;
  cudaError_t e = ensure_smem_attr(dgk::stage_lo4_kernel<MODE>, L::SMEM, attr);
  if (e != cudaSuccess) return e;
  const int ntiles = (A.e_end - A.e_begin + L::T - 1) / L::T;
  if (ntiles <= 0) return cudaSuccess;
  dgk::LoOp<1> O;
  const dgb::RefElem& R = c->ref;
  for (int n = 0; n < 4; ++n) {
    for (int k = 0; k < 4; ++k) {
      O.v[(0 + k) * 4 + n] = -R.Dr[n * 4 + k];
      O.v[(4 + k) * 4 + n] = -R.Ds[n * 4 + k];
      O.v[(8 + k) * 4 + n] = -R.Dt[n * 4 + k];
    }
    for (int k = 0; k < 12; ++k) O.v[(12 + k) * 4 + n] = R.LIFT[n * 12 + k];
  }
  for (int i = 0; i < 12; ++i) O.fm[i] = R.Fmask[i];
  return launch_stage_kernel(dgk::stage_lo4_kernel<MODE>, stage_grid(ntiles, max_ctas), L::NT, L::SMEM, st, (DG_PDL >> 1) & 1, A, O);
}

template <int MODE>
cudaError_t launch_stage(const dg_ctx* c, const dgk::StageArgs& A, int max_ctas, cudaStream_t st) {
  const int N = c->N;
  switch (N) {
    case 1: return DG_LO4 ? launch_lo4<MODE>(c, A, max_ctas, st) : launch_ws_n<1, MODE>(A, max_ctas, st);
    case 2: return launch_ws_n<2, MODE>(A, max_ctas, st);
    case 3: return launch_ws_n<3, MODE>(A, max_ctas, st);
    case 4: return launch_ws_n<4, MODE>(A, max_ctas, st);
    case 5: return launch_ho_n<5, MODE>(A, max_ctas, st);
    case 6: return launch_ho_n<6, MODE>(A, max_ctas, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_pack(dg_ctx* c, cudaStream_t st) {
  if (c->nsend == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t total = c->nsend * 5 * c->Nfp;
  const int grid = int(std::min<int64_t>((total + threads - 1) / threads, 8 * num_sms()));
  const double* Q = c->dQ[c->cur];
  switch (c->N) {
#define PACK(NN) case NN: dgk::pack_kernel<NN><<<grid, threads, 0, st>>>(Q, c->dselem, c->dsface, c->dtbl + 2 * 96 * c->Nfp, c->dsend, c->nsend); break;
    PACK(1) PACK(2) PACK(3) PACK(4) PACK(5) PACK(6)
#undef PACK
  }
  ++c->launches;
  return cudaGetLastError();
}

// operator tables uploaded to the workspace: DMMA B fragments (nodal) or the modal tables
const std::vector<double>& op_host(const dg_ctx* c) { return c->scheme == DG_SCHEME_MODAL ? c->modal_cat : c->opfrag; }

template <int P, int MODE>
cudaError_t launch_modal_p(const dgk::StageArgs& A, int max_ctas, cudaStream_t st) {
  using W = dgk::MW<P>;
  static uint64_t attr = 0;
  cudaError_t e = ensure_smem_attr(dgk::modal_warp_kernel<P, MODE>, W::SMEM, attr);
  if (e != cudaSuccess) return e;
  const int nel = A.e_end - A.e_begin;
  if (nel <= 0) return cudaSuccess;
  int grid = std::min((nel + W::WPC * W::EPW - 1) / (W::WPC * W::EPW), 8 * num_sms());
  if (max_ctas > 0) grid = std::min(grid, max_ctas);
  dgk::modal_warp_kernel<P, MODE><<<grid, W::NT, W::SMEM, st>>>(A);
  return cudaGetLastError();
}

// the modal tile kernel (modal.cuh): one persistent CTA per SM
template <int P, int MODE>
cudaError_t launch_modal_tile_p(const dgk::StageArgs& A, int max_ctas, cudaStream_t st) {
  using W = dgk::MT<P>;
  static uint64_t attr = 0;
  cudaError_t e = ensure_smem_attr(dgk::modal_tile_kernel<P, MODE>, W::SMEM, attr);
  if (e != cudaSuccess) return e;
  const int nel = A.e_end - A.e_begin;
  if (nel <= 0) return cudaSuccess;
  dgk::modal_tile_kernel<P, MODE><<<stage_grid((nel + W::EB - 1) / W::EB, max_ctas), W::NT, W::SMEM, st>>>(A);
  return cudaGetLastError();
}

// p = 1: four lanes per element on TMA-streamed tiles (lo.cuh modal_lo4_kernel); DG_MODAL_LO4 = 0
// keeps the tile kernel
#ifndef DG_MODAL_LO4
#define DG_MODAL_LO4 1
#endif
template <int MODE>
cudaError_t launch_modal_lo4(const dgk::StageArgs& A, int max_ctas, cudaStream_t st) {
  using L = dgk::ML4;
  static uint64_t attr = 0;
  cudaError_t e = ensure_smem_attr(dgk::modal_lo4_kernel<MODE>, L::SMEM, attr);
  if (e != cudaSuccess) return e;
  const int ntiles = (A.e_end - A.e_begin + L::T - 1) / L::T;
  if (ntiles <= 0) return cudaSuccess;
  return launch_stage_kernel(dgk::modal_lo4_kernel<MODE>, stage_grid(ntiles, max_ctas), L::NT, L::SMEM, st, (DG_PDL >> 1) & 1, A);
}

#ifndef DG_MODAL_TILE
#define DG_MODAL_TILE 1
#endif
template <int MODE>
cudaError_t launch_modal(int P, const dgk::StageArgs& A, int max_ctas, cudaStream_t st) {
  if (DG_MODAL_LO4 && P == 1) return launch_modal_lo4<MODE>(A, max_ctas, st);
  if (DG_MODAL_TILE) {
    switch (P) {
      case 1: return launch_modal_tile_p<1, MODE>(A, max_ctas, st);
      case 2: return launch_modal_tile_p<2, MODE>(A, max_ctas, st);
      case 3: return launch_modal_tile_p<3, MODE>(A, max_ctas, st);
    }
    return cudaErrorInvalidValue;
  }
  switch (P) {
    case 1: return launch_modal_p<1, MODE>(A, max_ctas, st);
    case 2: return launch_modal_p<2, MODE>(A, max_ctas, st);
    case 3: return launch_modal_p<3, MODE>(A, max_ctas, st);
  }
  return cudaErrorInvalidValue;
}

// per element and field: out = Mat in (Mat = V^-1: nodal -> modal; V: modal -> nodal)
cudaError_t modal_convert(dg_ctx* c, const double* in, double* out, bool to_modal, cudaStream_t st) {
  const int64_t n = c->K * 5 * c->Np;
  const int threads = 256;
  const int P = c->N;
  const size_t off = to_modal ? size_t(c->modal_cat.size() - size_t(c->Np) * c->Np)
                              : size_t(c->modal_cat.size() - 2 * size_t(c->Np) * c->Np);
  (void)P;
  dgk::modal_convert_kernel<<<int((n + threads - 1) / threads), threads, 0, st>>>(in, out, c->dop + off, c->K, c->Np);
  ++c->launches;
  return cudaGetLastError();
}

cudaError_t launch_sensors(dg_ctx* c, double* out, cudaStream_t st) {
  const int threads = 256, grid = (c->nsens * 32 + threads - 1) / threads;
  dgk::sensor_kernel<<<grid, threads, 0, st>>>(c->dQ[c->cur], c->dsel, c->dsw, c->nsens, c->Np, c->gamma, out);
  ++c->launches;
  return cudaGetLastError();
}

dgk::StageArgs base_args(dg_ctx* c, double t) {
  dgk::StageArgs A;
  std::memset(&A, 0, sizeof(A));
  A.Qin = c->dQ[c->cur];
  A.Qout = c->dQ[c->cur ^ 1];
  A.res = c->dres;
  A.geo = c->dgeo;
  A.nbr = c->dnbr;
  A.code = c->dcode;
  A.pub = c->dpub;
  A.recv = c->drecv;
  A.op = c->dop;
  A.tbl = c->dtbl;
  A.tblf = c->dtbl + 96 * c->Nfp;
  A.fmask = c->dtbl + 2 * 96 * c->Nfp;
  A.mtid = c->dmtid;
  A.flag = c->dflag;
  A.gid = c->dgid;
  A.Kpub = int(c->K);
  A.gamma = c->gamma;
  A.t = t;
  for (int i = 0; i < 5; ++i) A.qinf[i] = c->q_inf[i];
  // inflow ghost constants (reading A24): ambient state = q_inf (validated when used)
  A.in_p0 = c->qinf_valid ? c->pref : 1.0;
  A.in_rho0 = c->qinf_valid ? c->q_inf[0] : 1.4;
  A.in_c0 = std::sqrt(c->gamma * A.in_p0 / A.in_rho0);
  A.in_amp = c->inflow_half_amplitude * A.in_p0;
  A.in_omega = c->inflow_alpha * c->inflow_time_scale;
  A.lambda_mode = c->lambda_mode;
  A.skip = DG_DEBUG_SKIP;   // compile-time (0 in product builds)
  A.trace = reinterpret_cast<unsigned long long*>(c->dscratch);
  A.pref = c->pref;
  return A;
}

void set_range(dg_ctx* c, dgk::StageArgs& A, int which) {
  A.e_begin = (which & 1) ? 0 : int(c->K_int);
  A.e_end = (which & 2) ? int(c->K) : int(c->K_int);
}

dg_status need_bound(dg_ctx* c) {
  if (!c) return set_err(c, DG_EARG, "ctx is NULL");
  if (!c->ws) return set_err(c, DG_ESTATE, "no workspace bound");
  return DG_OK;
}

dg_status halo_exchange(dg_ctx* c, cudaStream_t st) {
  if (c->nparts == 1 || c->peers.empty()) return DG_OK;
  if (!c->comm) return set_err(c, DG_ESTATE, "nparts > 1 needs dg_comm_init (or the dg_stage_* driver)");
  CUDA_TRY(c, launch_pack(c, st));
  cudaStream_t cs = static_cast<cudaStream_t>(c->comm_stream);
  CUDA_TRY(c, cudaEventRecord(static_cast<cudaEvent_t>(c->ev_packed), st));
  CUDA_TRY(c, cudaStreamWaitEvent(cs, static_cast<cudaEvent_t>(c->ev_packed), 0));
  const size_t rec = size_t(5) * c->Nfp;
  ncclComm_t comm = static_cast<ncclComm_t>(c->comm);
  NCCL_TRY(c, ncclGroupStart());
  for (const dg_peer& p : c->peers) {
    if (p.nsend) NCCL_TRY(c, ncclSend(c->dsend + p.send_off * rec, p.nsend * rec, ncclDouble, p.rank, comm, cs));
    if (p.nrecv) NCCL_TRY(c, ncclRecv(c->drecv + p.recv_off * rec, p.nrecv * rec, ncclDouble, p.rank, comm, cs));
  }
  NCCL_TRY(c, ncclGroupEnd());
  CUDA_TRY(c, cudaEventRecord(static_cast<cudaEvent_t>(c->ev_recvd), cs));
  return DG_OK;
}

// grid cap of a launch: the interior launch of a partitioned step (which == 1, halo in flight)
// leaves nccl_ctas SMs free, so NCCL's send/recv kernel runs beside it instead of queueing
// behind the persistent CTAs (they hold every SM's registers and shared memory until they finish)
int launch_cap(const dg_ctx* c, int which) {
  int cap = c->max_ctas;
  if (which == 1 && c->comm && c->nccl_ctas > 0) {
    const int free_cap = std::max(1, num_sms() - c->nccl_ctas);
    cap = cap > 0 ? std::min(cap, free_cap) : free_cap;
  }
  return cap;
}

dg_status compute_stage(dg_ctx* c, int s, double dt, int which, cudaStream_t st) {
  double a, b, cc;
  coeffs(c, s, a, b, cc);
  dgk::StageArgs A = base_args(c, c->t + cc * dt);
  A.a = a;
  A.b = b;
  A.dt = dt;
  set_range(c, A, which);
  if (A.e_end > A.e_begin) {
    const int cap = launch_cap(c, which);
    CUDA_TRY(c, c->scheme == DG_SCHEME_MODAL ? launch_modal<dgk::MODE_UPDATE>(c->N, A, cap, st)
                                             : launch_stage<dgk::MODE_UPDATE>(c, A, cap, st));
    ++c->launches;
  }
  return DG_OK;
}

}  // namespace

extern "C" {

const char* dg_last_error(const dg_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

dg_status dg_mesh_create(const dg_mesh_desc* desc, int rank, dg_ctx** out) {
  if (!out) return set_err(nullptr, DG_EARG, "out is NULL");
  *out = nullptr;
  dg_ctx* c = new dg_ctx();
  dg_status st = dgb::build_ctx(desc, rank, c);
  if (st != DG_OK) {
    g_err = c->err;
    delete c;
    return st;
  }
  *out = c;
  return DG_OK;
}

void dg_destroy(dg_ctx* c) {
  if (!c) return;
  for (void*& g : c->graph_exec)
    if (g) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(g));
  if (c->capture_stream) cudaStreamDestroy(static_cast<cudaStream_t>(c->capture_stream));
  if (c->comm) ncclCommDestroy(static_cast<ncclComm_t>(c->comm));
  if (c->comm_stream) cudaStreamDestroy(static_cast<cudaStream_t>(c->comm_stream));
  if (c->ev_packed) cudaEventDestroy(static_cast<cudaEvent_t>(c->ev_packed));
  if (c->ev_recvd) cudaEventDestroy(static_cast<cudaEvent_t>(c->ev_recvd));
  delete c;
}

dg_status dg_sizes(const dg_ctx* c, int64_t* k, int* np, int* nfp) {
  if (!c) return set_err(nullptr, DG_EARG, "ctx is NULL");
  if (k) *k = c->K;
  if (np) *np = c->Np;
  if (nfp) *nfp = c->Nfp;
  return DG_OK;
}

size_t dg_workspace_bytes(const dg_ctx* c) {
  if (!c) return 0;
  const size_t st = size_t(c->K) * 5 * c->Np * 8;
  size_t b = 0;
  b += 2 * align256(st);                                           // Q ping-pong
  b += align256(st);                                               // res
  b += align256(st);                                               // staging
  b += align256(size_t(c->K) * dgk::GEO * 8);                      // geo
  b += align256(size_t(c->K) * 16) + align256(size_t(c->K) * 4) + align256(size_t(c->K) * 4) + align256(size_t(c->K) * 8);
  b += align256(op_host(c).size() * 8) + align256(2 * 96 * c->Nfp + 4 * c->Nfp);
  if (!c->mtid.empty()) b += align256(c->mtid.size());                // modal face-point table ids
  const size_t rec = size_t(5) * c->Nfp * 8;
  b += align256(c->nsend * rec) + align256(c->nrecv * rec) + align256(c->nsend * 4) + align256(c->nsend);
  b += align256(64) + align256(4096 * 8);
  b += align256(size_t(DG_MAX_SENSORS) * c->Np * 8) + align256(size_t(DG_MAX_SENSORS) * 4);   // sensors
  return b;
}

dg_status dg_memory_report(const dg_ctx* c, size_t bytes[7]) {
  if (!c || !bytes) return set_err(nullptr, DG_EARG, "NULL argument");
  const size_t st = size_t(c->K) * 5 * c->Np * 8;
  const size_t rec = size_t(5) * c->Nfp * 8;
  bytes[0] = 2 * st;
  bytes[1] = st;
  bytes[2] = st;
  bytes[3] = size_t(c->K) * dgk::GEO * 8;
  bytes[4] = size_t(c->K) * (16 + 4 + 4 + 8) + c->mtid.size();
  bytes[5] = op_host(c).size() * 8 + 2 * 96 * c->Nfp + 4 * c->Nfp + size_t(DG_MAX_SENSORS) * (c->Np * 8 + 4);
  bytes[6] = (c->nsend + c->nrecv) * rec + c->nsend * 5;
  return DG_OK;
}

static dg_status upload_sensors(dg_ctx* c, cudaStream_t st);

dg_status dg_bind_workspace(dg_ctx* c, void* dptr, size_t nbytes, void* stream) {
  if (!c || !dptr) return set_err(c, DG_EARG, "NULL argument");
  if (nbytes < dg_workspace_bytes(c)) return set_err(c, DG_EARG, "workspace too small");
  if (reinterpret_cast<uintptr_t>(dptr) % 256) return set_err(c, DG_EARG, "workspace must be 256-byte aligned");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* p = static_cast<char*>(dptr);
  auto take = [&](size_t n) {
    char* r = p;
    p += align256(n);
    return r;
  };
  const size_t stb = size_t(c->K) * 5 * c->Np * 8;
  c->dQ[0] = reinterpret_cast<double*>(take(stb));
  c->dQ[1] = reinterpret_cast<double*>(take(stb));
  c->dres = reinterpret_cast<double*>(take(stb));
  c->dstage = reinterpret_cast<double*>(take(stb));
  c->dgeo = reinterpret_cast<double*>(take(size_t(c->K) * dgk::GEO * 8));
  c->dnbr = reinterpret_cast<int32_t*>(take(size_t(c->K) * 16));
  c->dcode = reinterpret_cast<uint8_t*>(take(size_t(c->K) * 4));
  c->dpub = reinterpret_cast<int32_t*>(take(size_t(c->K) * 4));
  c->dgid = reinterpret_cast<int64_t*>(take(size_t(c->K) * 8));
  c->dop = reinterpret_cast<double*>(take(op_host(c).size() * 8));
  c->dtbl = reinterpret_cast<uint8_t*>(take(2 * 96 * c->Nfp + 4 * c->Nfp));
  c->dmtid = c->mtid.empty() ? nullptr : reinterpret_cast<uint8_t*>(take(c->mtid.size()));
  const size_t rec = size_t(5) * c->Nfp * 8;
  c->dsend = reinterpret_cast<double*>(take(c->nsend * rec));
  c->drecv = reinterpret_cast<double*>(take(c->nrecv * rec));
  c->dselem = reinterpret_cast<int32_t*>(take(c->nsend * 4));
  c->dsface = reinterpret_cast<uint8_t*>(take(c->nsend));
  c->dflag = reinterpret_cast<int*>(take(64));
  c->dscratch = reinterpret_cast<double*>(take(4096 * 8));
  c->dsw = reinterpret_cast<double*>(take(size_t(DG_MAX_SENSORS) * c->Np * 8));
  c->dsel = reinterpret_cast<int32_t*>(take(size_t(DG_MAX_SENSORS) * 4));
  for (void*& g : c->graph_exec)   // captured steps point into the previous workspace
    if (g) {
      cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(g));
      g = nullptr;
    }
  c->rec_buf = nullptr;
  c->ws = dptr;
  c->ws_bytes = nbytes;
  dg_memory_report(c, c->cat_bytes);
  CUDA_TRY(c, cudaMemcpyAsync(c->dgeo, c->geo.data(), c->geo.size() * 8, cudaMemcpyHostToDevice, st));
  CUDA_TRY(c, cudaMemcpyAsync(c->dnbr, c->nbr.data(), c->nbr.size() * 4, cudaMemcpyHostToDevice, st));
  CUDA_TRY(c, cudaMemcpyAsync(c->dcode, c->code.data(), c->code.size(), cudaMemcpyHostToDevice, st));
  CUDA_TRY(c, cudaMemcpyAsync(c->dpub, c->pub.data(), c->pub.size() * 4, cudaMemcpyHostToDevice, st));
  CUDA_TRY(c, cudaMemcpyAsync(c->dgid, c->gid.data(), c->gid.size() * 8, cudaMemcpyHostToDevice, st));
  CUDA_TRY(c, cudaMemcpyAsync(c->dop, op_host(c).data(), op_host(c).size() * 8, cudaMemcpyHostToDevice, st));
  std::vector<uint8_t>& tb = c->tbl;  // concatenated tables live until the copy completes (synced below)
  std::vector<uint8_t> all(tb);
  all.insert(all.end(), c->tblf.begin(), c->tblf.end());
  all.insert(all.end(), c->fmask8.begin(), c->fmask8.end());
  CUDA_TRY(c, cudaMemcpyAsync(c->dtbl, all.data(), all.size(), cudaMemcpyHostToDevice, st));
  if (c->dmtid) CUDA_TRY(c, cudaMemcpyAsync(c->dmtid, c->mtid.data(), c->mtid.size(), cudaMemcpyHostToDevice, st));
  if (c->nsend) {
    CUDA_TRY(c, cudaMemcpyAsync(c->dselem, c->send_elem.data(), c->nsend * 4, cudaMemcpyHostToDevice, st));
    CUDA_TRY(c, cudaMemcpyAsync(c->dsface, c->send_face.data(), c->nsend, cudaMemcpyHostToDevice, st));
  }
  CUDA_TRY(c, cudaMemsetAsync(c->dflag, 0, 64, st));
  CUDA_TRY(c, cudaMemsetAsync(c->dQ[0], 0, 3 * align256(stb), st));
  if (c->nsens > 0) {   // sensors placed before the workspace was bound
    dg_status e = upload_sensors(c, st);
    if (e) return e;
  }
  CUDA_TRY(c, cudaStreamSynchronize(st));   // host vectors above are pageable / temporaries
  return DG_OK;
}

dg_status dg_get_nodes(const dg_ctx* c, double* x, double* y, double* z) {
  if (!c || !x || !y || !z) return set_err(nullptr, DG_EARG, "NULL argument");
  const size_t n = size_t(c->K) * c->Np;
  std::memcpy(x, c->xyz.data(), n * 8);
  std::memcpy(y, c->xyz.data() + n, n * 8);
  std::memcpy(z, c->xyz.data() + 2 * n, n * 8);
  return DG_OK;
}

dg_status dg_set_state(dg_ctx* c, const double* rho, const double* mx, const double* my, const double* mz,
                       const double* E, int on_device, double t, void* stream) {
  dg_status s0 = need_bound(c);
  if (s0) return s0;
  if (!rho || !mx || !my || !mz || !E) return set_err(c, DG_EARG, "NULL state array");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t n = size_t(c->K) * c->Np;
  const double* src[5] = {rho, mx, my, mz, E};
  for (int q = 0; q < 5; ++q)
    CUDA_TRY(c, cudaMemcpyAsync(c->dstage + q * n, src[q], n * 8, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  const int threads = 256;
  const int grid = int(std::min<int64_t>((int64_t(n) * 5 + threads - 1) / threads, 16 * num_sms()));
  c->cur = 0;
  dgk::to_internal_kernel<<<grid, threads, 0, st>>>(c->dstage, c->dpub, c->dQ[0], c->dres, c->K, c->Np);
  ++c->launches;
  CUDA_TRY(c, cudaGetLastError());
  if (c->scheme == DG_SCHEME_MODAL) {   // nodal values -> coefficients (interpolation, reading A23)
    CUDA_TRY(c, modal_convert(c, c->dQ[0], c->dQ[1], true, st));
    c->cur = 1;
  }
  CUDA_TRY(c, cudaMemsetAsync(c->dflag, 0, 64, st));
  c->t = t;
  c->state_set = true;
  c->steps_done = 0;
  return DG_OK;
}

dg_status dg_get_state(dg_ctx* c, double* rho, double* mx, double* my, double* mz, double* E, int on_device,
                       void* stream) {
  dg_status s0 = need_bound(c);
  if (s0) return s0;
  if (!rho || !mx || !my || !mz || !E) return set_err(c, DG_EARG, "NULL state array");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t n = size_t(c->K) * c->Np;
  const int threads = 256;
  const int grid = int(std::min<int64_t>((int64_t(n) * 5 + threads - 1) / threads, 16 * num_sms()));
  const double* src = c->dQ[c->cur];
  if (c->scheme == DG_SCHEME_MODAL) {   // coefficients -> nodal values, in the spare state buffer
    CUDA_TRY(c, modal_convert(c, c->dQ[c->cur], c->dQ[c->cur ^ 1], false, st));
    src = c->dQ[c->cur ^ 1];
  }
  dgk::to_public_kernel<<<grid, threads, 0, st>>>(src, c->dpub, c->dstage, c->K, c->Np);
  ++c->launches;
  CUDA_TRY(c, cudaGetLastError());
  double* dst[5] = {rho, mx, my, mz, E};
  for (int q = 0; q < 5; ++q)
    CUDA_TRY(c, cudaMemcpyAsync(dst[q], c->dstage + q * n, n * 8, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
  return DG_OK;
}

dg_status dg_get_time(const dg_ctx* c, double* t) {
  if (!c || !t) return set_err(nullptr, DG_EARG, "NULL argument");
  *t = c->t;
  return DG_OK;
}

dg_status dg_spectrum(const double* x, int64_t n, int64_t m, double* amp, double* db, void* stream) {
  if (!x || !amp || !db) return set_err(nullptr, DG_EARG, "dg_spectrum: NULL pointer");
  if (n < 2 || m < 1 || m > 65535) return set_err(nullptr, DG_EARG, "dg_spectrum: need n >= 2 and 1 <= m <= 65535");
  const int64_t nb = n / 2 + 1;
  const int wpb = 8;
  const dim3 grid(unsigned((nb + wpb - 1) / wpb), unsigned(m));
  dgk::spectrum_kernel<<<grid, 32 * wpb, 0, static_cast<cudaStream_t>(stream)>>>(x, n, m, amp, db);
  CUDA_TRY(nullptr, cudaGetLastError());
  return DG_OK;
}

dg_status dg_set_nccl_ctas(dg_ctx* c, int nctas) {
  if (!c) return set_err(c, DG_EARG, "ctx is NULL");
  if (nctas < 0 || nctas > 64) return set_err(c, DG_EARG, "nctas must be in [0, 64]");
  if (c->comm) return set_err(c, DG_ESTATE, "dg_set_nccl_ctas must precede dg_comm_init");
  c->nccl_ctas = nctas;
  return DG_OK;
}

dg_status dg_set_max_ctas(dg_ctx* c, int max_ctas) {
  if (!c) return set_err(nullptr, DG_EARG, "ctx is NULL");
  if (max_ctas < 0) return set_err(c, DG_EARG, "max_ctas must be >= 0");
  if (c->max_ctas != max_ctas)
    for (void*& g : c->graph_exec)   // captured steps carry the old grid
      if (g) {
        cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(g));
        g = nullptr;
      }
  c->max_ctas = max_ctas;
  return DG_OK;
}

#define DG_STR2(x) #x
#define DG_STR(x) DG_STR2(x)
const char* dg_build_info(void) {
  return "arch=sm_100a;DG_TRACE=" DG_STR(DG_TRACE) ";DG_DEBUG_SKIP=" DG_STR(DG_DEBUG_SKIP)
#ifdef DG_WS_PW
         ";DG_WS_PW=" DG_STR(DG_WS_PW)
#endif
#ifdef DG_WS_CW
         ";DG_WS_CW=" DG_STR(DG_WS_CW)
#endif
#ifdef DG_WS_EB
         ";DG_WS_EB=" DG_STR(DG_WS_EB)
#endif
#ifdef DG_KUNROLL
         ";DG_KUNROLL=" DG_STR(DG_KUNROLL)
#endif
#ifdef DG_NEWTON2
         ";DG_NEWTON2=1"
#endif
#ifdef DG_SKIP_VOL
         ";DG_SKIP_VOL=" DG_STR(DG_SKIP_VOL)
#endif
#ifdef DG_WS_IOW
         ";DG_WS_IOW=" DG_STR(DG_WS_IOW)
#endif
#ifdef DG_HO_KC
         ";DG_HO_KC=" DG_STR(DG_HO_KC)
#endif
#ifdef DG_HO_SLOTS
         ";DG_HO_SLOTS=" DG_STR(DG_HO_SLOTS)
#endif
         ";DG_SDF=" DG_STR(DG_SDF) ";DG_HO_SDF=" DG_STR(DG_HO_SDF);
}

dg_status dg_check(dg_ctx* c, void* stream) {
  dg_status s0 = need_bound(c);
  if (s0) return s0;
  int h[2] = {0, 0};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CUDA_TRY(c, cudaMemcpyAsync(h, c->dflag, 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(c, cudaStreamSynchronize(st));
  if (h[0]) {
    char buf[160];
    std::snprintf(buf, sizeof(buf), "invalid state (rho<=0, p<=0 or non-finite) in element %d at t=%.17g", h[1], c->t);
    return set_err(c, DG_EBLOWUP, buf);
  }
  return DG_OK;
}

dg_status dg_rhs_compute(dg_ctx* c, double t, double* out, int which, void* stream) {
  dg_status s0 = need_bound(c);
  if (s0) return s0;
  if (!out) return set_err(c, DG_EARG, "out is NULL");
  if (!c->state_set) return set_err(c, DG_ESTATE, "state not set");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  dgk::StageArgs A = base_args(c, t);
  A.out = out;
  set_range(c, A, which);
  if (A.e_end > A.e_begin) {
    CUDA_TRY(c, c->scheme == DG_SCHEME_MODAL ? launch_modal<dgk::MODE_RHS>(c->N, A, launch_cap(c, which), st)
                                             : launch_stage<dgk::MODE_RHS>(c, A, launch_cap(c, which), st));
    ++c->launches;
  }
  return DG_OK;
}

dg_status dg_rhs(dg_ctx* c, double t, double* out, void* stream) {
  dg_status s0 = need_bound(c);
  if (s0) return s0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (c->nparts > 1 && !c->peers.empty()) {
    dg_status e = halo_exchange(c, st);
    if (e) return e;
    e = dg_rhs_compute(c, t, out, 1, stream);
    if (e) return e;
    CUDA_TRY(c, cudaStreamWaitEvent(st, static_cast<cudaEvent_t>(c->ev_recvd), 0));
    return dg_rhs_compute(c, t, out, 2, stream);
  }
  return dg_rhs_compute(c, t, out, 3, stream);
}

dg_status dg_halo_exchange(dg_ctx* c, void* stream) {
  dg_status s0 = need_bound(c);
  if (s0) return s0;
  if (!c->state_set) return set_err(c, DG_ESTATE, "state not set");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (c->nparts == 1 || c->peers.empty()) return DG_OK;
  dg_status e = halo_exchange(c, st);
  if (e) return e;
  CUDA_TRY(c, cudaStreamWaitEvent(st, static_cast<cudaEvent_t>(c->ev_recvd), 0));
  return DG_OK;
}

dg_status dg_stage_pack(dg_ctx* c, void* stream) {
  dg_status s0 = need_bound(c);
  if (s0) return s0;
  CUDA_TRY(c, launch_pack(c, static_cast<cudaStream_t>(stream)));
  return DG_OK;
}

dg_status dg_stage_compute(dg_ctx* c, int s, double dt, int which, void* stream) {
  dg_status s0 = need_bound(c);
  if (s0) return s0;
  if (!c->state_set) return set_err(c, DG_ESTATE, "state not set");
  if (s < 0 || s >= nstages(c)) return set_err(c, DG_EARG, "stage index out of range");
  return compute_stage(c, s, dt, which, static_cast<cudaStream_t>(stream));
}

dg_status dg_stage_finish(dg_ctx* c, int s, double dt) {
  dg_status s0 = need_bound(c);
  if (s0) return s0;
  c->cur ^= 1;
  if (s == nstages(c) - 1) {
    c->t += dt;
    ++c->steps_done;
  }
  return DG_OK;
}

dg_status dg_rk_step(dg_ctx* c, double dt, int nsteps, void* stream) {
  dg_status s0 = need_bound(c);
  if (s0) return s0;
  if (!c->state_set) return set_err(c, DG_ESTATE, "state not set");
  if (nsteps < 0 || !std::isfinite(dt)) return set_err(c, DG_EARG, "bad dt or nsteps");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool multi = c->nparts > 1 && !c->peers.empty();
  // single partition, no time-dependent boundary, no per-step host work: replay one captured
  // step (its stage launches) as a CUDA graph; the first step of a new dt runs eagerly
  const bool graphable = !multi && !c->has_inflow && !c->rec_buf && c->check_every == 0 &&
                         std::getenv("DG_NO_GRAPHS") == nullptr;
  if (graphable && c->graph_dt != dt) {
    for (void*& g : c->graph_exec)
      if (g) {
        cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(g));
        g = nullptr;
      }
    c->graph_dt = dt;
  }
  int n = 0;
  if (graphable && nsteps > 1) {
    if (!c->graph_exec[0] && !c->graph_exec[1]) {   // eager first step: sets kernel attributes
      for (int s = 0; s < nstages(c); ++s) {
        dg_status e = compute_stage(c, s, dt, 3, st);
        if (e) return e;
        dg_stage_finish(c, s, dt);
      }
      n = 1;
    }
    for (; n < nsteps; ++n) {
      cudaGraphExec_t& ex = reinterpret_cast<cudaGraphExec_t&>(c->graph_exec[c->cur]);
      if (!ex) {
        if (!c->capture_stream) {
          cudaStream_t cs;
          CUDA_TRY(c, cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
          c->capture_stream = cs;
        }
        cudaStream_t cs = static_cast<cudaStream_t>(c->capture_stream);
        const int cur0 = c->cur;
        const double t0 = c->t;
        const int64_t l0 = c->launches, s0n = c->steps_done;
        CUDA_TRY(c, cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        for (int s = 0; s < nstages(c); ++s) {
          dg_status e = compute_stage(c, s, dt, 3, cs);
          if (e) {
            cudaGraph_t gbad = nullptr;
            cudaStreamEndCapture(cs, &gbad);
            if (gbad) cudaGraphDestroy(gbad);
            return e;
          }
          dg_stage_finish(c, s, dt);
        }
        cudaGraph_t gr;
        CUDA_TRY(c, cudaStreamEndCapture(cs, &gr));
        CUDA_TRY(c, cudaGraphInstantiate(&ex, gr, 0));
        cudaGraphDestroy(gr);
        c->cur = cur0;   // capturing ran nothing: restore the step state
        c->t = t0;
        c->steps_done = s0n;
        c->launches = l0;
      }
      CUDA_TRY(c, cudaGraphLaunch(ex, st));
      for (int s = 0; s < nstages(c); ++s) dg_stage_finish(c, s, dt);
      c->launches += nstages(c);
    }
    return DG_OK;
  }
  for (; n < nsteps; ++n) {
    for (int s = 0; s < nstages(c); ++s) {
      if (multi) {
        dg_status e = halo_exchange(c, st);
        if (e) return e;
        e = compute_stage(c, s, dt, 1, st);
        if (e) return e;
        CUDA_TRY(c, cudaStreamWaitEvent(st, static_cast<cudaEvent_t>(c->ev_recvd), 0));
        e = compute_stage(c, s, dt, 2, st);
        if (e) return e;
      } else {
        dg_status e = compute_stage(c, s, dt, 3, st);
        if (e) return e;
      }
      dg_stage_finish(c, s, dt);
    }
    if (c->rec_buf && c->nsens > 0 && c->rec_count < c->rec_cap) {
      CUDA_TRY(c, launch_sensors(c, c->rec_buf + c->rec_count * c->nsens * 6, st));
      ++c->rec_count;
    }
    if (c->check_every > 0 && (c->steps_done % c->check_every) == 0) {
      dg_status e = dg_check(c, stream);
      if (e) return e;
    }
  }
  return DG_OK;
}

dg_status dg_stable_dt(dg_ctx* c, double cfl, double* dt, void* stream) {
  dg_status s0 = need_bound(c);
  if (s0) return s0;
  if (!dt || !(cfl > 0)) return set_err(c, DG_EARG, "bad argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t nn = c->K * c->Np;
  const int threads = 256;
  const int grid = int(std::min<int64_t>((nn + threads - 1) / threads, 4096));
  const double* q = c->dQ[c->cur];
  if (c->scheme == DG_SCHEME_MODAL) {   // wave speeds at the nodes
    CUDA_TRY(c, modal_convert(c, c->dQ[c->cur], c->dQ[c->cur ^ 1], false, st));
    q = c->dQ[c->cur ^ 1];
  }
  dgk::max_speed_kernel<<<grid, threads, 0, st>>>(q, nn, c->Np, c->gamma, c->dscratch);
  ++c->launches;
  CUDA_TRY(c, cudaGetLastError());
  std::vector<double> part(grid);
  CUDA_TRY(c, cudaMemcpyAsync(part.data(), c->dscratch, grid * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(c, cudaStreamSynchronize(st));
  double lam = 0;
  for (double v : part) lam = std::max(lam, v);
  double hmin = *std::min_element(c->h.begin(), c->h.end());
  if (!(lam > 0) || !std::isfinite(lam)) return set_err(c, DG_EBLOWUP, "non-finite wave speed in stable_dt");
  *dt = cfl * hmin / ((c->N + 1) * (c->N + 1) * lam);
  return DG_OK;
}

dg_status dg_nccl_get_unique_id(void* out128) {
  if (!out128) return set_err(nullptr, DG_EARG, "NULL argument");
  ncclUniqueId id;
  NCCL_TRY(nullptr, ncclGetUniqueId(&id));
  std::memcpy(out128, &id, sizeof(id));
  return DG_OK;
}

dg_status dg_comm_init(dg_ctx* c, const void* uid, int nranks) {
  if (!c || !uid) return set_err(c, DG_EARG, "NULL argument");
  if (nranks != c->nparts) return set_err(c, DG_EARG, "nranks must equal nparts");
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  ncclComm_t comm;
  // NCCL's kernels are capped at DG_NCCL_CTAS (default 2) CTAs; the interior stage launch leaves
  // that many SMs free (launch_cap), and the communication stream has the highest priority
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  const int nctas = c->nccl_ctas;   // dg_set_nccl_ctas, default 2
  if (nctas > 0) {
    cfg.minCTAs = 1;
    cfg.maxCTAs = nctas;
  }
  NCCL_TRY(c, ncclCommInitRankConfig(&comm, nranks, id, c->rank, &cfg));
  c->comm = comm;
  cudaStream_t cs;
  int prio_lo = 0, prio_hi = 0;
  CUDA_TRY(c, cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  CUDA_TRY(c, cudaStreamCreateWithPriority(&cs, cudaStreamNonBlocking, prio_hi));
  c->comm_stream = cs;
  cudaEvent_t e1, e2;
  CUDA_TRY(c, cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
  CUDA_TRY(c, cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
  c->ev_packed = e1;
  c->ev_recvd = e2;
  return DG_OK;
}

dg_status dg_halo_info(const dg_ctx* c, int* npeers, int64_t* nsend, int64_t* nrecv) {
  if (!c) return set_err(nullptr, DG_EARG, "ctx is NULL");
  if (npeers) *npeers = int(c->peers.size());
  if (nsend) *nsend = c->nsend;
  if (nrecv) *nrecv = c->nrecv;
  return DG_OK;
}

dg_status dg_halo_peer(const dg_ctx* c, int p, int* rank, int64_t* send_off, int64_t* nsend, int64_t* recv_off,
                       int64_t* nrecv) {
  if (!c || p < 0 || p >= int(c->peers.size())) return set_err(nullptr, DG_EARG, "bad peer index");
  const dg_peer& q = c->peers[p];
  if (rank) *rank = q.rank;
  if (send_off) *send_off = q.send_off;
  if (nsend) *nsend = q.nsend;
  if (recv_off) *recv_off = q.recv_off;
  if (nrecv) *nrecv = q.nrecv;
  return DG_OK;
}

dg_status dg_halo_buffers(const dg_ctx* c, double** send, double** recv) {
  if (!c || !c->ws) return set_err(nullptr, DG_ESTATE, "no workspace bound");
  if (send) *send = c->dsend;
  if (recv) *recv = c->drecv;
  return DG_OK;
}

dg_status dg_halo_records(const dg_ctx* c, int64_t* send_gid, int8_t* send_face, int64_t* recv_gid, int8_t* recv_face) {
  if (!c) return set_err(nullptr, DG_EARG, "ctx is NULL");
  for (int64_t s = 0; s < c->nsend; ++s) {
    if (send_gid) send_gid[s] = c->gid[c->send_elem[s]];
    if (send_face) send_face[s] = int8_t(c->send_face[s]);
  }
  for (int64_t g = 0; g < c->nrecv; ++g) {
    if (recv_gid) recv_gid[g] = c->recv_gid[g];
    if (recv_face) recv_face[g] = int8_t(c->recv_face[g]);
  }
  return DG_OK;
}

dg_status dg_get_operators(const dg_ctx* c, double* r, double* s, double* t, double* Dr, double* Ds, double* Dt,
                           double* LIFT, int32_t* Fmask) {
  if (!c) return set_err(nullptr, DG_EARG, "ctx is NULL");
  const auto& R = c->ref;
  if (r) std::copy(R.r.begin(), R.r.end(), r);
  if (s) std::copy(R.s.begin(), R.s.end(), s);
  if (t) std::copy(R.t.begin(), R.t.end(), t);
  if (Dr) std::copy(R.Dr.begin(), R.Dr.end(), Dr);
  if (Ds) std::copy(R.Ds.begin(), R.Ds.end(), Ds);
  if (Dt) std::copy(R.Dt.begin(), R.Dt.end(), Dt);
  if (LIFT) std::copy(R.LIFT.begin(), R.LIFT.end(), LIFT);
  if (Fmask)
    for (size_t i = 0; i < R.Fmask.size(); ++i) Fmask[i] = R.Fmask[i];
  return DG_OK;
}

dg_status dg_get_maps(const dg_ctx* c, int64_t* vmapM, int64_t* vmapP) {
  if (!c || !vmapM || !vmapP) return set_err(nullptr, DG_EARG, "NULL argument");
  const int Np = c->Np, Nfp = c->Nfp;
  // reported in PUBLIC element order
  for (int64_t l = 0; l < c->K; ++l) {
    const int64_t p = c->pub[l];
    for (int f = 0; f < 4; ++f) {
      const int code = c->code[l * 4 + f];
      for (int i = 0; i < Nfp; ++i) {
        const int64_t m = p * Np + c->ref.Fmask[f * Nfp + i];
        const size_t o = (size_t(p) * 4 + f) * Nfp + i;
        vmapM[o] = m;
        if (code >= dgk::CODE_BC) {
          vmapP[o] = m;
        } else if (code >= dgk::CODE_GHOST) {
          const int j = c->tblf[(f * 24 + code - dgk::CODE_GHOST) * Nfp + i];
          vmapP[o] = -1 - (int64_t(c->nbr[l * 4 + f]) * Nfp + j);
        } else {
          vmapP[o] = int64_t(c->pub[c->nbr[l * 4 + f]]) * Np + c->tbl[(f * 24 + code) * Nfp + i];
        }
      }
    }
  }
  return DG_OK;
}

dg_status dg_get_geometry(const dg_ctx* c, double* J, double* rx9, double* n12, double* fs4) {
  if (!c) return set_err(nullptr, DG_EARG, "ctx is NULL");
  for (int64_t l = 0; l < c->K; ++l) {
    const int64_t p = c->pub[l];
    const double* G = &c->geo[l * dgk::GEO];
    if (J) J[p] = c->J[l];
    for (int i = 0; i < 9; ++i)
      if (rx9) rx9[p * 9 + i] = G[i];
    for (int f = 0; f < 4; ++f) {
      for (int q = 0; q < 3; ++q)
        if (n12) n12[p * 12 + 3 * f + q] = G[9 + 4 * f + q];
      if (fs4) fs4[p * 4 + f] = G[9 + 4 * f + 3];
    }
  }
  return DG_OK;
}

int64_t dg_launch_count(const dg_ctx* c) { return c ? c->launches : 0; }

static dg_status upload_sensors(dg_ctx* c, cudaStream_t st) {
  if (c->nsens == 0 || !c->ws) return DG_OK;
  CUDA_TRY(c, cudaMemcpyAsync(c->dsw, c->sens_w.data(), c->sens_w.size() * 8, cudaMemcpyHostToDevice, st));
  CUDA_TRY(c, cudaMemcpyAsync(c->dsel, c->sens_elem.data(), size_t(c->nsens) * 4, cudaMemcpyHostToDevice, st));
  CUDA_TRY(c, cudaStreamSynchronize(st));   // the host vectors may change on the next call
  return DG_OK;
}

dg_status dg_sensors_set(dg_ctx* c, int n, const double* xyz, int32_t* elem_out, void* stream) {
  if (!c) return set_err(nullptr, DG_EARG, "ctx is NULL");
  if (n < 0 || n > DG_MAX_SENSORS || (n > 0 && !xyz)) return set_err(c, DG_EARG, "sensor count out of range or NULL points");
  const int Np = c->Np;
  const int64_t K = c->K;
  // reference corner nodes (v1..v4) of the node set
  int corner[4] = {-1, -1, -1, -1};
  const double cr[4][3] = {{-1, -1, -1}, {1, -1, -1}, {-1, 1, -1}, {-1, -1, 1}};
  for (int v = 0; v < 4; ++v)
    for (int q = 0; q < Np; ++q)
      if (std::fabs(c->ref.r[q] - cr[v][0]) < 1e-12 && std::fabs(c->ref.s[q] - cr[v][1]) < 1e-12 &&
          std::fabs(c->ref.t[q] - cr[v][2]) < 1e-12)
        corner[v] = q;
  for (int v = 0; v < 4; ++v)
    if (corner[v] < 0) return set_err(c, DG_EARG, "reference corner node not found");
  std::vector<int32_t> el(n, -1);
  std::vector<int64_t> best_gid(n, INT64_MAX);
  std::vector<double> rst(3 * size_t(n), 0.0);
  const double tol = 1e-10;
  const size_t KN = size_t(K) * Np;
  for (int64_t l = 0; l < K; ++l) {
    const int64_t pb = c->pub[l];
    double vx[4][3];
    for (int v = 0; v < 4; ++v)
      for (int d = 0; d < 3; ++d) vx[v][d] = c->xyz[d * KN + size_t(pb) * Np + corner[v]];
    double lo[3], hi[3];
    for (int d = 0; d < 3; ++d) {
      lo[d] = std::min(std::min(vx[0][d], vx[1][d]), std::min(vx[2][d], vx[3][d]));
      hi[d] = std::max(std::max(vx[0][d], vx[1][d]), std::max(vx[2][d], vx[3][d]));
    }
    const double pad = 1e-9 * (hi[0] - lo[0] + hi[1] - lo[1] + hi[2] - lo[2]);
    const double* G = &c->geo[size_t(l) * 25];
    for (int i = 0; i < n; ++i) {
      const double* x = xyz + 3 * size_t(i);
      if (x[0] < lo[0] - pad || x[0] > hi[0] + pad || x[1] < lo[1] - pad || x[1] > hi[1] + pad ||
          x[2] < lo[2] - pad || x[2] > hi[2] + pad)
        continue;
      const double d0 = x[0] - vx[0][0], d1 = x[1] - vx[0][1], d2 = x[2] - vx[0][2];
      // (1+r, 1+s, 1+t) = (grad r, grad s, grad t) . (x - v1)
      const double r1 = G[0] * d0 + G[1] * d1 + G[2] * d2;
      const double s1 = G[3] * d0 + G[4] * d1 + G[5] * d2;
      const double t1 = G[6] * d0 + G[7] * d1 + G[8] * d2;
      const double lam[4] = {1.0 - (r1 + s1 + t1) / 2, r1 / 2, s1 / 2, t1 / 2};   // barycentrics of v1..v4
      if (lam[0] < -tol || lam[1] < -tol || lam[2] < -tol || lam[3] < -tol) continue;
      if (c->gid[l] < best_gid[i]) {
        best_gid[i] = c->gid[l];
        el[i] = int32_t(l);
        rst[3 * i] = r1 - 1.0;
        rst[3 * i + 1] = s1 - 1.0;
        rst[3 * i + 2] = t1 - 1.0;
      }
    }
  }
  c->nsens = n;
  c->sens_elem = el;
  c->sens_w.assign(size_t(n) * Np, 0.0);
  for (int i = 0; i < n; ++i) {
    if (el[i] >= 0) {
      double* w = &c->sens_w[size_t(i) * Np];
      dgb::interp_weights(c->ref, rst[3 * i], rst[3 * i + 1], rst[3 * i + 2], w);
      if (c->scheme == DG_SCHEME_MODAL) {   // the state is coefficients: weights psi_m = sum_n l_n V_nm
        std::vector<double> l(w, w + Np);
        for (int mm = 0; mm < Np; ++mm) {
          double acc = 0;
          for (int nn = 0; nn < Np; ++nn) acc += l[nn] * c->modal.V[size_t(nn) * Np + mm];
          w[mm] = acc;
        }
      }
    }
    if (elem_out) elem_out[i] = el[i] >= 0 ? c->pub[el[i]] : -1;
  }
  dg_status e = upload_sensors(c, static_cast<cudaStream_t>(stream));   // or at dg_bind_workspace
  if (e) return e;
  c->rec_buf = nullptr;
  c->rec_cap = c->rec_count = 0;
  return DG_OK;
}

dg_status dg_sensors_sample(dg_ctx* c, double* out, int on_device, void* stream) {
  dg_status s0 = need_bound(c);
  if (s0) return s0;
  if (!out) return set_err(c, DG_EARG, "NULL output");
  if (!c->state_set) return set_err(c, DG_ESTATE, "state not set");
  if (c->nsens == 0) return DG_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* dst = on_device ? out : c->dscratch;   // scratch holds 4096 doubles >= 256 x 6
  CUDA_TRY(c, launch_sensors(c, dst, st));
  if (!on_device) {
    CUDA_TRY(c, cudaMemcpyAsync(out, dst, size_t(c->nsens) * 6 * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(c, cudaStreamSynchronize(st));
  }
  return DG_OK;
}

dg_status dg_sensors_record(dg_ctx* c, double* dbuf, int64_t capacity) {
  dg_status s0 = need_bound(c);
  if (s0) return s0;
  if (dbuf && capacity <= 0) return set_err(c, DG_EARG, "capacity must be positive");
  c->rec_buf = dbuf;
  c->rec_cap = dbuf ? capacity : 0;
  c->rec_count = 0;
  return DG_OK;
}

int64_t dg_sensors_recorded(const dg_ctx* c) { return c ? c->rec_count : 0; }

// Debug only (DG_TRACE builds): copy the phase-timestamp scratch of the last stage launch.
dg_status dg_debug_trace(const dg_ctx* c, unsigned long long* out, int n) {
  if (!c || !c->ws || !out || n <= 0 || n > 4096) return set_err(nullptr, DG_EARG, "bad argument");
  CUDA_TRY(nullptr, cudaMemcpy(out, c->dscratch, size_t(n) * 8, cudaMemcpyDeviceToHost));
  return DG_OK;
}

}  // extern "C"
