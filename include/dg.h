/*
 * dg.h -- C ABI of the B200-native nodal-DG Euler RHS + explicit RK stage library
 * (libdg_b200.so).  Hot path of arXiv:1710.03887 (J. Resch), Appendix A:
 * the discontinuous Galerkin discretisation of the 3D
 * compressible Euler equations, Eq. 1-2, on affine tetrahedra,
 * with the pass-through, reflective wall and inflow
 * boundary conditions and explicit Runge-Kutta time stepping
 * (P:41).  Citation key and the readings of garbled/ambiguous passages:
 * DESIGN.md ("Readings").
 *
 * Conventions (all part of the ABI):
 *  - order N >= 1 (N <= DG_MAX_ORDER), Np = (N+1)(N+2)(N+3)/6 nodes per element,
 *    Nfp = (N+1)(N+2)/2 nodes per face.
 *  - reference tetrahedron {r,s,t >= -1, r+s+t <= -1}; local vertices
 *    v1=(-1,-1,-1), v2=(1,-1,-1), v3=(-1,1,-1), v4=(-1,-1,1) are EToV[k][0..3].
 *  - local faces: f0 = (v1 v2 v3) [t=-1], f1 = (v1 v2 v4) [s=-1],
 *    f2 = (v2 v3 v4) [r+s+t=-1], f3 = (v1 v3 v4) [r=-1].
 *  - nodes: warp & blend (alpha = 0) on the reference tet, ordered by the
 *    equispaced lattice index (i,j,k): k (t) outermost, j (s), i (r) innermost.
 *  - state: conserved variables (rho, rho u, rho v, rho w, E) of Eq. 1.
 *    Public layout is field-major [5][K_local][Np] (five arrays of K_local*Np),
 *    element order = this rank's elements in ascending global id.
 *  - all arithmetic is IEEE fp64.
 *  - every device operation is ordered on the caller's CUDA stream (passed as
 *    void* = cudaStream_t).  A ctx is not thread-safe.  The library never
 *    calls cudaMalloc: the caller binds one device workspace.
 *
 * Errors: every call returns a dg_status.  dg_last_error(ctx) (or
 * dg_last_error(NULL) for failures without a ctx) gives a message that names
 * the element and the time for invalid-state errors.
 */
#ifndef DG_B200_H
#define DG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DG_MAX_ORDER 6
#define DG_MAX_SENSORS 256

typedef enum dg_status {
  DG_OK = 0,
  DG_EARG = 2,          /* bad argument or configuration (SPEC S:624 exit 2)             */
  DG_EMESH = 3,         /* non-manifold face, J <= 0 with given connectivity, bad/missing  */
                        /* boundary tag, asymmetric EToE/EToF, unmatched face nodes */
  DG_EBLOWUP = 4,       /* rho <= 0, p <= 0 or non-finite state (exit 4)    */
  DG_ECUDA = 5,         /* CUDA runtime error                                             */
  DG_ENCCL = 6,         /* NCCL error                                                     */
  DG_EUNSUPPORTED = 7,  /* valid request this build does not implement                    */
  DG_ESTATE = 8         /* call out of order (e.g. no workspace bound yet)                */
} dg_status;

/* boundary tags per element face */
enum { DG_BC_INTERIOR = 0, DG_BC_WALL = 1, DG_BC_PASSTHROUGH = 2, DG_BC_INFLOW = 3 };

/* time integrators ("RK2"; BASELINE.json configs: LSERK4) */
enum { DG_RK_LSERK4 = 0, DG_RK_HEUN = 1 };

/* spatial schemes: nodal collocation (default) or the paper's own modal
 * scheme with Gauss quadrature (orders 1-3, one partition) */
enum { DG_SCHEME_NODAL = 0, DG_SCHEME_MODAL = 1 };

typedef struct dg_ctx dg_ctx;

typedef struct dg_mesh_desc {
  int order;                 /* N                                                           */
  int64_t nv;                /* number of vertices                                          */
  const double* vxyz;        /* nv x 3, row-major, host                                     */
  int64_t k;                 /* number of tetrahedra (whole mesh, all ranks)                */
  const int64_t* etov;       /* k x 4, 0-based vertex ids, host                             */
  const int64_t* etoe;       /* k x 4 neighbour element, or NULL = derive by face hashing   */
  const int8_t* etof;        /* k x 4 neighbour local face (NULL iff etoe is NULL)          */
                             /* a boundary face points at itself (etoe=k, etof=f); periodic */
                             /* faces pair across the domain (a pure translation)           */
  const int8_t* bc;          /* k x 4 boundary tag (DG_BC_*); 0 exactly on paired faces     */
  double gamma;              /* ratio of specific heats (~1.4)                       */
  double q_inf[5];           /* pass-through ghost state (Eq. 3)                 */
  const int32_t* part;       /* k entries -> owning rank, or NULL = single partition        */
  int nparts;                /* number of ranks in `part` (1 if part is NULL)               */
  int lambda_mode;           /* LLF wave-speed bound: 0 = max over the face's nodes          */
                             /* (default), 1 = per node (reading A4)               */
  int check_every;           /* dg_rk_step checks the blow-up flag every n steps (0 = never) */
  int rk_scheme;             /* DG_RK_LSERK4 (default) or DG_RK_HEUN                         */
  double inflow_alpha;       /* pulse angular frequency of the inflow BC: rad per */
                             /* physical second; <= 0 = the paper's 565 (A24)     */
  int scheme;                /* DG_SCHEME_NODAL (default) or DG_SCHEME_MODAL: the state of   */
                             /* dg_set_state / dg_get_state / dg_rhs stays nodal values at   */
                             /* the dg_get_nodes points; internally the modal scheme steps   */
                             /* orthonormal coefficients (interpolation c = V^-1 u, A23)     */
  double inflow_time_scale;  /* physical seconds per scaled time unit for the inflow pulse:  */
                             /* p1 uses cos(alpha * time_scale * t); <= 0 = 2.915e-5 (1 cm / */
                             /* 343 m/s); 1.0 makes alpha rad per scaled unit    */
  double inflow_half_amplitude; /* a of p1 = p0 (1 + a - a cos(...)); <= 0 = 0.05 */
} dg_mesh_desc;
/* Inflow ghost (Eqs. 5-7) in the units of q_inf: p0 = p(q_inf), rho0 = q_inf[0],
 * c0 = sqrt(gamma p0 / rho0); rho = rho0 (p/p0)^(1/gamma) (Eq. 6 with C = rho0 p0^(-1/gamma),
 * = gamma at the paper's p0 = 1, rho0 = 1.4), u = (p - p0)/(rho0 c0) (Eq. 5), v = w = 0.
 * q_inf must be a valid state (finite, rho > 0, p > 0) when the mesh has pass-through or
 * inflow faces (else DG_EARG); otherwise it is unused. */

/* Build a context for `rank` (0 <= rank < nparts): validate the mesh, fix or
 * reject orientation (a J <= 0 tet is repaired by swapping its local vertices
 * 2 and 3 only when etoe == NULL, else DG_EMESH; the repair moves the tags of
 * its faces f1 and f3 with the vertex sets the swap exchanges, so bc stays in
 * the caller's face numbering), derive/check connectivity, build the reference
 * operators (fp64, orthonormal Jacobi basis), geometric factors, trace pairing
 * and this rank's halo lists.  Host arrays are only read during the call; the
 * caller keeps ownership.  No device work. */
dg_status dg_mesh_create(const dg_mesh_desc* desc, int rank, dg_ctx** out);
void dg_destroy(dg_ctx* ctx);
const char* dg_last_error(const dg_ctx* ctx);

/* sizes of this rank's problem */
dg_status dg_sizes(const dg_ctx* ctx, int64_t* k_local, int* np, int* nfp);

/* Device workspace: the caller allocates dg_workspace_bytes() bytes (256-byte
 * aligned) and keeps them alive until dg_destroy.  Binding uploads operators,
 * geometry and connectivity on `stream`. */
size_t dg_workspace_bytes(const dg_ctx* ctx);
dg_status dg_bind_workspace(dg_ctx* ctx, void* dptr, size_t nbytes, void* stream);
/* per-category bytes, categories: 0 state (Q x2), 1 residual, 2 staging,
 * 3 geometry, 4 connectivity, 5 operators, 6 halo; SPEC memory_report */
dg_status dg_memory_report(const dg_ctx* ctx, size_t bytes[7]);

/* Physical node coordinates, host arrays of K_local*Np each (element-major, ABI node order). */
dg_status dg_get_nodes(const dg_ctx* ctx, double* x, double* y, double* z);

/* Copy in the state (five arrays of K_local*Np; host if on_device == 0, else
 * device pointers), zero the RK residual and set t.  Host arrays should be
 * pinned for an asynchronous copy.  The copy is complete when `stream` is. */
dg_status dg_set_state(dg_ctx* ctx, const double* rho, const double* mx, const double* my,
                       const double* mz, const double* E, int on_device, double t, void* stream);
/* Mirror of dg_set_state: copy the current state out (host or device). */
dg_status dg_get_state(dg_ctx* ctx, double* rho, double* mx, double* my, double* mz, double* E,
                       int on_device, void* stream);
dg_status dg_get_time(const dg_ctx* ctx, double* t);

/* f(Q, t) of eq:ode: writes 5*K_local*Np fp64 to the DEVICE buffer
 * `out`, public layout [5][K_local][Np].  Does not modify the state.  With
 * nparts > 1 it exchanges face traces (NCCL) first. */
dg_status dg_rhs(dg_ctx* ctx, double t, double* out, void* stream);

/* nsteps explicit RK steps of size dt (caller-supplied, so both sides of a
 * parity run use the same dt): per stage s, res = a_s res + dt f(Q, t + c_s dt),
 * Q += b_s res.  t advances by nsteps*dt.  The blow-up flag is read back every
 * check_every steps (0 = never) and raises DG_EBLOWUP with the element id. */
dg_status dg_rk_step(dg_ctx* ctx, double dt, int nsteps, void* stream);

/* Cap the number of CTAs (one per SM) of the persistent stage kernels; 0 = one per SM of the
 * device (default).  A smaller grid makes every CTA walk more element tiles -- the tests use it to
 * reach the pipelined steady state on small meshes -- and leaves SMs free for concurrent work
 * (e.g. the NCCL halo kernels, see dg_rk_step).  Results do not depend on it. */
dg_status dg_set_max_ctas(dg_ctx* ctx, int max_ctas);

/* One-sided amplitude spectra of m uniformly sampled pressure records (SURVEY §8(f) N4,
 * DESIGN.md reading A22; Fig. 5 and §3): per record the mean is removed,
 * X_k = sum_j x_j e^{-2 pi i jk/n}, amp_k = 2|X_k|/n (|X_k|/n at k = 0 and, for even n, at
 * k = n/2), db_k = 20 log10(amp_k) floored at -200 dB (re 1 scaled pressure unit).
 * x: DEVICE array n x m row-major (sample j of record r at x[j*m + r], e.g. a
 * dg_sensors_record buffer column); amp, db: DEVICE arrays (n/2+1) x m, caller-owned.
 * Stream-ordered on `stream`; no ctx (errors via dg_last_error(NULL)): DG_EARG for NULL
 * pointers, n < 2, m < 1 or m > 65535; DG_ECUDA on a launch failure. */
dg_status dg_spectrum(const double* x, int64_t n, int64_t m, double* amp, double* db, void* stream);

/* Compile-time configuration of this build ("key=value;..."), for benchmark records. */
const char* dg_build_info(void);

/* Synchronously read the device blow-up flag (DG_EBLOWUP if set). */
dg_status dg_check(dg_ctx* ctx, void* stream);

/* Host helper (S:299-307 reading, A10): dt = cfl * min_k h_k /
 * ((N+1)^2 * max_nodes(|u| + c)) with h_k = 3 V_k / max face area, from the
 * current state (synchronous).  Local to this rank; allreduce-min across ranks
 * is the caller's (or dg_rk_step's) concern. */
dg_status dg_stable_dt(dg_ctx* ctx, double cfl, double* dt, void* stream);

/* ---- multi-GPU (element partition) ------------------------- */
/* NCCL unique id (128 bytes) for rank 0 to broadcast. */
dg_status dg_nccl_get_unique_id(void* out128);
/* Initialise this ctx's NCCL communicator (nranks must equal desc->nparts).  The communicator
 * is created with maxCTAs = the dg_set_nccl_ctas value (default 2) and a highest-priority
 * stream; while the halo is in flight the interior stage launch of dg_rk_step / dg_rhs
 * leaves that many SMs free, so the exchange overlaps the interior work (
 * DG needs only face-neighbour data).  DG_ENCCL on an NCCL failure. */
dg_status dg_comm_init(dg_ctx* ctx, const void* unique_id128, int nranks);
/* SMs reserved for NCCL's kernel during the interior launch (0 = none: the halo kernel then
 * waits for free SMs); must precede dg_comm_init, nctas in [0, 64], else DG_EARG / DG_ESTATE. */
dg_status dg_set_nccl_ctas(dg_ctx* ctx, int nctas);

/* Halo description for transport-agnostic use (tests, custom transports):
 * per peer p in [0, npeers): its rank, and the face-trace records sent to and
 * received from it.  A record is 5*Nfp doubles (field-major, sender's face
 * node order); send/recv buffers are device arrays inside the workspace. */
dg_status dg_halo_info(const dg_ctx* ctx, int* npeers, int64_t* nsend_total, int64_t* nrecv_total);
dg_status dg_halo_peer(const dg_ctx* ctx, int p, int* rank, int64_t* send_off, int64_t* nsend,
                       int64_t* recv_off, int64_t* nrecv);
dg_status dg_halo_buffers(const dg_ctx* ctx, double** send, double** recv);
/* Host description of the halo records (tests, custom transports): for send
 * record s, the sender's global element id and local face; for receive record
 * g, the remote (sender) global element id and face.  Arrays of nsend / nrecv. */
dg_status dg_halo_records(const dg_ctx* ctx, int64_t* send_gid, int8_t* send_face, int64_t* recv_gid,
                          int8_t* recv_face);
/* Stage-level driver for custom transports: pack this rank's partition-face
 * traces of the current state into the send buffer; then, once the recv
 * buffer holds the peers' records, run stage s (0-based) of the RK scheme on
 * the interior (which & 1) and/or boundary (which & 2) elements; then finish
 * the stage (swap state buffers, advance t after the last stage). */
dg_status dg_stage_pack(dg_ctx* ctx, void* stream);
/* Pack + NCCL exchange of the current state's partition-face traces (what every stage of
 * dg_rk_step does before its boundary launch); the receive buffer is complete when `stream`
 * reaches its current point.  No-op on one partition.  Needs dg_comm_init.  For timing the
 * halo alone (bench.py) and for custom stage drivers. */
dg_status dg_halo_exchange(dg_ctx* ctx, void* stream);
dg_status dg_stage_compute(dg_ctx* ctx, int s, double dt, int which, void* stream);
dg_status dg_stage_finish(dg_ctx* ctx, int s, double dt);
/* same, for one RHS evaluation into `out` (public layout) */
dg_status dg_rhs_compute(dg_ctx* ctx, double t, double* out, int which, void* stream);

/* ---- point sensors (Table 2: "the generated
 * pressure was sampled at various positions throughout the computational domain")
 * dg_sensors_set: n <= DG_MAX_SENSORS points xyz (host, n x 3 row-major, copied).
 * Each point is located in this rank's elements (barycentric test with tolerance
 * 1e-10; on a shared face/edge/vertex the element with the smallest global id
 * wins) and the nodal interpolation weights l_i(r,s,t) of its element are
 * computed on the host and uploaded.  elem_out (host, n; may be NULL) receives
 * the public element index on this rank or -1 when the point lies on another
 * rank or outside the mesh.  Replaces any earlier set; stops recording.
 * dg_sensors_sample: the state at every sensor -- the conserved variables
 * interpolated at the point and p = (gamma-1)(E - |m|^2/(2 rho)) from them
 * (reading A21) -- as n rows (rho, m_x, m_y, m_z, E, p) into out
 * (device pointer if on_device, else host); rows of sensors not on this rank
 * are NaN.  Stream-ordered after the stepping calls on the same stream.
 * dg_sensors_record: from now on every step of dg_rk_step appends one sample
 * (n x 6 doubles) to the caller's device buffer dbuf (capacity samples; the
 * caller keeps ownership); NULL stops recording.  dg_sensors_recorded returns
 * the number of samples written so far. */
dg_status dg_sensors_set(dg_ctx* ctx, int n, const double* xyz, int32_t* elem_out, void* stream);
dg_status dg_sensors_sample(dg_ctx* ctx, double* out, int on_device, void* stream);
dg_status dg_sensors_record(dg_ctx* ctx, double* dbuf, int64_t capacity);
int64_t dg_sensors_recorded(const dg_ctx* ctx);

/* ---- introspection (tests) ------------------------------------------------ */
/* Reference operators: r,s,t (Np), Dr/Ds/Dt (Np x Np, row-major), LIFT
 * (Np x 4 Nfp, row-major, column block f in Fmask_f order), Fmask (4 x Nfp). */
dg_status dg_get_operators(const dg_ctx* ctx, double* r, double* s, double* t, double* Dr,
                           double* Ds, double* Dt, double* LIFT, int32_t* Fmask);
/* Trace maps in the oracle's convention: for each local element k, face f,
 * face node i: vmapM = k*Np + Fmask_f[i], vmapP = neighbour's node (local
 * index, or -1-g for the g-th received ghost record's node when the
 * neighbour is remote; = vmapM on a physical boundary).  Arrays K_local*4*Nfp. */
dg_status dg_get_maps(const dg_ctx* ctx, int64_t* vmapM, int64_t* vmapP);
/* Geometric factors per local element: J, (r,s,t)_(x,y,z) 9 values row-major,
 * normals 4x3, Fscale 4. */
dg_status dg_get_geometry(const dg_ctx* ctx, double* J, double* rx9, double* n12, double* fscale4);
/* Counts of kernel launches issued by this ctx since creation (gpu_launches). */
int64_t dg_launch_count(const dg_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* DG_B200_H */
