// Internal context of libdg_b200 (one per rank and device).
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/dg.h"
#include "refelem.h"

struct dg_peer {
  int rank;
  int64_t send_off, nsend, recv_off, nrecv;
};

struct dg_ctx {
  // ---- configuration
  int N = 0, Np = 0, Nfp = 0;
  int rank = 0, nparts = 1;
  double gamma = 1.4;
  double q_inf[5] = {1.4, 0, 0, 0, 2.5};
  int lambda_mode = 0, check_every = 0, rk_scheme = DG_RK_LSERK4;
  double inflow_alpha = 565.0, inflow_time_scale = 2.915e-5, inflow_half_amplitude = 0.05;
  double pref = 0.0;              // ambient pressure p(q_inf) subtracted from the fluxes (A14), 0 if unused
  bool qinf_valid = false;
  int max_ctas = 0;               // stage-kernel grid cap (0 = one CTA per SM)
  int nccl_ctas = 2;              // SMs left free for NCCL's kernel while the interior launch runs (P > 1)
  int scheme = DG_SCHEME_NODAL;
  dgb::RefElem ref;
  dgb::ModalTables modal;           // scheme == DG_SCHEME_MODAL
  std::vector<double> modal_cat;    // concatenated tables (kernels.cuh MS<P> offsets)

  // ---- this rank's elements, internal order: interior first, then partition-boundary
  int64_t K = 0, K_int = 0;
  std::vector<int64_t> gid;      // internal -> global element id
  std::vector<int32_t> pub;      // internal -> public index (rank's elements, ascending gid)
  std::vector<double> geo;       // K x 25: (r,s,t)_(x,y,z) row-major, then 4 x (n, Fscale)
  std::vector<double> J, h;      // K
  std::vector<int32_t> nbr;      // K x 4: neighbour internal index / halo record / -1
  std::vector<uint8_t> code;     // K x 4: f2*6+sigma | 32+f2*6+sigma | 64+tag
  std::vector<uint8_t> tbl, tblf, fmask8;   // neighbour node tables (uint8)
  std::vector<uint8_t> mtid;     // modal scheme: K x 4 x (own, neighbour) face-point table ids
  std::vector<double> xyz;       // 3 x K x Np node coordinates, PUBLIC element order
  std::vector<double> opfrag;    // B-fragment operator for the DMMA contraction

  // ---- halo
  std::vector<dg_peer> peers;
  std::vector<int32_t> send_elem;   // per send record: internal element
  std::vector<uint8_t> send_face;   // per send record: local face
  std::vector<int64_t> recv_gid;    // per recv record: sender's global element
  std::vector<uint8_t> recv_face;   // per recv record: sender's face
  int64_t nsend = 0, nrecv = 0;

  // ---- device workspace
  void* ws = nullptr;
  size_t ws_bytes = 0;
  double* dQ[2] = {nullptr, nullptr};
  double* dres = nullptr;
  double* dstage = nullptr;
  double* dgeo = nullptr;
  int32_t* dnbr = nullptr;
  uint8_t* dcode = nullptr;
  int32_t* dpub = nullptr;
  int64_t* dgid = nullptr;
  double* dop = nullptr;
  uint8_t* dtbl = nullptr;     // tbl | tblf | fmask
  uint8_t* dmtid = nullptr;    // K x 8 (modal scheme)
  double* dsend = nullptr;
  double* drecv = nullptr;
  int32_t* dselem = nullptr;
  uint8_t* dsface = nullptr;
  int* dflag = nullptr;
  double* dscratch = nullptr;
  size_t cat_bytes[7] = {0, 0, 0, 0, 0, 0, 0};

  // ---- point sensors
  int nsens = 0;
  std::vector<int32_t> sens_elem;   // internal element or -1 (not on this rank)
  std::vector<double> sens_w;       // nsens x Np interpolation weights
  double* dsw = nullptr;            // device: DG_MAX_SENSORS x Np weights
  int32_t* dsel = nullptr;          // device: DG_MAX_SENSORS elements
  double* rec_buf = nullptr;        // caller's device buffer, rec_cap x nsens x 6
  int64_t rec_cap = 0, rec_count = 0;

  // ---- run state
  int cur = 0;          // which dQ holds the current state
  double t = 0.0;
  bool state_set = false;
  int64_t steps_done = 0;
  int64_t launches = 0;
  std::string err;

  // ---- CUDA graphs of one RK step (single partition): [start buffer cur] for the cached dt
  void* graph_exec[2] = {nullptr, nullptr};
  void* capture_stream = nullptr;
  double graph_dt = 0.0;
  bool has_inflow = false;

  // ---- NCCL (opaque to keep nccl.h out of the host translation units)
  void* comm = nullptr;
  void* comm_stream = nullptr;
  void* ev_packed = nullptr;
  void* ev_recvd = nullptr;
};

namespace dgb {
// host-side mesh processing (mesh.cpp); fills everything up to the halo lists
dg_status build_ctx(const dg_mesh_desc* d, int rank, dg_ctx* c);
}
