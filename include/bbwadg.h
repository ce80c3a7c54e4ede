/*
 * bbwadg.h -- C ABI of the B200-native BBWADG hot path (libbbwadg.so).
 *
 * Bernstein-Bezier weight-adjusted DG (Guo & Chan, arXiv 1808.08645) for the
 * 3D acoustic wave equation in heterogeneous media.  Citations "P:n" are
 * PAPER.md line numbers (section / equation named); "S:n" SPEC.md lines.
 *
 * What one RK stage computes ("three kernels", fused here):
 *   volume   r_p = -div u, r_u = -grad p            (Eq. WADGform P:141-142,
 *                                                     sparse Bernstein derivative P:264)
 *   surface  + sum_f (J_f/J) L^f F   with the penalty fluxes of Eq. sdf
 *             and the factorised lift L^f = E^f_L L_0
 *   WADG     dp/dt = P^{N+M}_N (c^2_M * r_p)        (Bernstein product
 *            Eq. mcoeff; telescoping projection Eq. telescope)
 *   LSRK     res = a_s res + dt rhs;  Q = Q + b_s res   (Carpenter-Kennedy)
 *
 * Conventions (DESIGN.md "Readings" R1-R23 where the paper is silent):
 *   - weight multiplied in the WADG update is c^2 (R1);
 *   - fields per element: (p, u_x, u_y, u_z); state layout Q[K][4][Np],
 *     element-major, Np = (N+1)(N+2)(N+3)/6, contiguous per element;
 *   - Bernstein coefficient order ("canonical", R19):
 *       for a3 in 0..N: for a2 in 0..N-a3: for a1 in 0..N-a3-a2: a0 = N-a1-a2-a3
 *     local vertex i of an element <-> barycentric lambda_i <-> exponent a_i;
 *   - face f is the face opposite local vertex f; neighbours are matched by
 *     global vertex ids (exact, no geometric tolerance);
 *   - boundary faces: pressure release, p+ = -p, u+ = u (R11);
 *   - penalties default tau_p = tau_u = 1 (R10).
 *
 * Ownership: the caller owns every host input; setup copies what it needs.
 * The context owns all device state (Q ping-pong buffers, residual, tables,
 * halo buffers, NCCL communicator).  Device pointers passed to rhs/wadg_apply/
 * set_state/get_state are caller-owned, must live on the context's device,
 * use the canonical layout and the context's dtype (double for BBWADG_F64,
 * float for BBWADG_F32).  All device work is ordered on the context's stream.
 * A context is not thread-safe, and its kernels must not run concurrently with
 * each other: the stage kernels take element batches from a per-context work
 * queue counter (device memory owned by the context, reset by each launch's
 * last CTA), so two stage launches of one context on different streams at the
 * same time would share it.  Stream-ordered use through this API never does.
 *
 * Tuning environment variables (read at setup; not needed in normal use):
 * BBWADG_BLOCKS_PER_SM=b lowers the persistent grid to b CTAs per SM;
 * BBWADG_FORCE_BLOCKS_PER_SM=b sets it regardless of the occupancy query;
 * BBWADG_PHASE_TIMING allocates per-phase cycle counters (timing builds);
 * BBWADG_NO_GRAPH disables the CUDA-graph replay of bbwadg_run.
 *
 * Errors: every call returns a bbwadg_status; nothing aborts or throws across
 * the ABI.  bbwadg_error_string(ctx) (or bbwadg_last_error() when no context
 * exists yet) returns the text of the last error.  Asynchronous CUDA faults
 * surface at the next synchronising call as BBWADG_ERR_CUDA.
 */
#ifndef BBWADG_H
#define BBWADG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BBWADG_MAX_N 9            /* supported degrees: 1 <= N <= 9, 0 <= M <= N */
#define BBWADG_NCCL_ID_BYTES 128

typedef struct bbwadg_ctx_s* bbwadg_ctx;

typedef enum {
  BBWADG_OK = 0,
  BBWADG_ERR_INVALID_ARG = 1,     /* null pointer, bad size, bad option */
  BBWADG_ERR_MESH = 2,            /* J <= 0, face shared by > 2 elements, bad vertex id */
  BBWADG_ERR_NONPOSITIVE_C2 = 3,  /* c^2_M <= 0 at a check point (R16/R23) */
  BBWADG_ERR_UNSUPPORTED = 4,     /* N/M out of range, dtype */
  BBWADG_ERR_CUDA = 5,
  BBWADG_ERR_NCCL = 6,
  BBWADG_ERR_NONFINITE = 7,       /* NaN/Inf in the state after bbwadg_run */
  BBWADG_ERR_OOM = 8,
  BBWADG_ERR_NO_DEVICE = 9
} bbwadg_status;

typedef enum { BBWADG_F64 = 0, BBWADG_F32 = 1 } bbwadg_dtype;

/* Affine tetrahedral mesh, host memory, read during setup only.
 * vertices [num_vertices][3] physical coordinates; elements [num_elements][4]
 * global vertex ids, positively oriented: det[X1-X0, X2-X0, X3-X0] > 0
 * (the orientation of the reference tetrahedron).  Elements with
 * J <= 0 are rejected, never reordered (c^2 coefficients are tied to the
 * caller's vertex order). */
typedef struct {
  int64_t num_vertices;
  const double* vertices;
  int64_t num_elements;
  const int64_t* elements;
} bbwadg_mesh;

typedef struct {
  int dtype;             /* bbwadg_dtype; default BBWADG_F64 */
  double tau_p, tau_u;   /* penalty parameters of Eq. sdf; default 1, 1 */
  int device;            /* CUDA device ordinal; default 0 */
  void* cuda_stream;     /* cudaStream_t to order all work on; NULL = the legacy default stream */
  int rank, world_size;  /* element-partitioned multi-GPU run; world_size 1 = single GPU */
  const void* nccl_unique_id; /* ncclUniqueId (128 bytes) from bbwadg_nccl_unique_id on rank 0,
                                 broadcast by the caller; required when world_size > 1 */
  int partition[3];      /* cut counts per axis for the recursive coordinate bisection
                            (product must equal world_size); {0,0,0} = automatic */
  int check_c2;          /* 1 (default): reject non-positive c^2_M at setup */
  int halo_transport;    /* partition faces (world_size > 1 or groups): 0 (default) = pack (p, u.n) per
                            face + NCCL send/recv (device copies in groups); 1 = PEER READS: the stage
                            kernel reads the owner partition's Q_in in place (same device: groups; other
                            processes / GPUs: CUDA IPC, bbwadg_ipc_get_handles / bbwadg_ipc_open_peer), no
                            pack, no collective, bitwise equal to the single-partition run */
  const int64_t* c2_gids; /* optional (multi-GPU memory): when non-NULL, c2_coeffs of bbwadg_setup holds
                             c2_rows rows, row i for global element c2_gids[i] (e.g. this rank's elements
                             from bbwadg_partition_plan); every element the rank owns must be present
                             (else BBWADG_ERR_INVALID_ARG).  NULL: c2_coeffs is [K][Mp] in global order */
  int64_t c2_rows;
  int reserved[4];
} bbwadg_options;

typedef struct {
  int64_t num_elements_global;   /* K */
  int64_t num_elements_local;    /* elements owned by this rank */
  int64_t num_interior_local;    /* local elements without off-rank neighbours (first in local order) */
  int64_t num_halo_faces;        /* faces whose neighbour lives on another rank */
  int N, M, Np, Mp, dtype, rank, world_size;
  const int64_t* global_ids;     /* [num_elements_local]: global element id of each local element
                                    (host memory owned by the ctx) */
  double algorithmic_bytes_per_stage;  /* minimum HBM bytes of one fused stage over the local
                                          elements */
  double flops_per_stage;              /* algorithmic flops of one stage over local elements */
  int kernels_per_stage;               /* kernel launches per RK stage */
  int64_t steps_taken;
  double time;
} bbwadg_info;

/* Fill defaults (F64, tau 1/1, device 0, cuda_stream NULL = the legacy default stream, single GPU, check_c2). */
void bbwadg_default_options(bbwadg_options* opts);

/* Build the context: validate and partition the mesh, compute geometric
 * factors, build per-(N,M) operator tables, upload everything to the device.
 *   c2_coeffs: host [K][Mp] degree-M Bernstein coefficients of c^2 per element
 *              (global element order), Mp = (M+1)(M+2)(M+3)/6; or, with
 *              opts->c2_gids, [c2_rows][Mp] rows for those global element ids only.
 * The state is zero after setup. */
bbwadg_status bbwadg_setup(const bbwadg_mesh* mesh, int N, int M, const double* c2_coeffs,
                           const bbwadg_options* opts, bbwadg_ctx* out);

/* State Q[K_local][4][Np] in local element order (global_ids gives the map;
 * identical to the global order when world_size == 1).  on_device = 1: Q is a
 * device pointer on the ctx's device; 0: host memory.  dtype = ctx dtype.
 * set_state also zeroes the LSRK residual. */
bbwadg_status bbwadg_set_state(bbwadg_ctx ctx, const void* Q, int on_device);
bbwadg_status bbwadg_get_state(bbwadg_ctx ctx, void* Q, int on_device);

/* Optional manufactured-solution source of the pressure equation:
 * g host [K][Np] (global order, double) with r_p += g * sin(pi t) before the
 * WADG projection (R17).  NULL removes it. */
bbwadg_status bbwadg_set_source(bbwadg_ctx ctx, const double* g);

/* dQ/dt of Eq. WADGform at time t for the device state Q_dev (local order):
 * dp/dt after the WADG update, du/dt = r_u.  Multi-GPU: exchanges the
 * partition-face traces of Q_dev first (collective over all ranks). */
bbwadg_status bbwadg_rhs(bbwadg_ctx ctx, const void* Q_dev, double t, void* dQdt_dev);

/* Test hook: out = P^{N+M}_N (c^2_M * r) per element, device
 * arrays [K_local][Np]. */
bbwadg_status bbwadg_wadg_apply(bbwadg_ctx ctx, const void* r_dev, void* out_dev);

/* One LSRK45 step (5 fused stages) of the context's state from t to t+dt. */
bbwadg_status bbwadg_step(bbwadg_ctx ctx, double t, double dt);

/* nsteps steps from t0; synchronises at the end and checks the state for
 * NaN/Inf (BBWADG_ERR_NONFINITE).  On single-partition contexts without a source
 * and nsteps >= 2 the step is replayed as a CUDA graph (5 stage launches captured
 * once per dt on a private stream ordered with the context's stream; bitwise equal
 * to bbwadg_step; environment variable BBWADG_NO_GRAPH disables it). */
bbwadg_status bbwadg_run(bbwadg_ctx ctx, double t0, double dt, int64_t nsteps);

/* Block until all work queued on the ctx's stream has finished. */
bbwadg_status bbwadg_synchronize(bbwadg_ctx ctx);

bbwadg_status bbwadg_query(bbwadg_ctx ctx, bbwadg_info* info);
const char* bbwadg_error_string(bbwadg_ctx ctx);
const char* bbwadg_last_error(void);
void bbwadg_destroy(bbwadg_ctx ctx);

/* ---- elastic BBWADG: velocity-stress elastic wave equation, Eq. ewave
 * (P:150-157), DG form with penalty fluxes P:198-206, matrix-weighted WADG update Eq. ewadg
 * with the isotropic C of P:185-195.  One fused kernel per RK stage (volume, surface, ten scalar
 * weight-adjusted applications, LSRK); R25-R28.
 *   rho_inv, lambda, mu: host [K][Mp] degree-M Bernstein coefficients of rho^-1 and the Lame
 *              parameters per element (global order); setup rejects rho^-1 <= 0, lambda + 2 mu <= 0
 *              or mu < 0 at the check points (opts->check_c2).
 *   opts:      tau_p is the stress penalty tau_sigma, tau_u the velocity penalty tau_v (the acoustic
 *              p <-> sigma, u <-> v correspondence); world_size must be 1; c2_gids unused.
 * The returned context uses the common calls with 9 fields: state Q[K][9][Np] with fields
 * (v_1, v_2, v_3, s11, s22, s33, s23, s13, s12) (Voigt order of the A_i rows);
 * bbwadg_rhs gives dQ/dt of Eq. ewadg; bbwadg_wadg_apply maps r[K][9][Np] to
 * (P_N(rho^-1 r_v), (I x M^-1) M_C r_sigma); step/run/get/set_state/query/destroy as above;
 * bbwadg_set_source and partition groups are not available (BBWADG_ERR_UNSUPPORTED /
 * BBWADG_ERR_INVALID_ARG).  Errors as for bbwadg_setup. */
bbwadg_status bbwadg_elastic_setup(const bbwadg_mesh* mesh, int N, int M, const double* rho_inv,
                                   const double* lambda, const double* mu, const bbwadg_options* opts,
                                   bbwadg_ctx* out);

/* ---- 2D triangles (2D experiments P:646-652): the acoustic
 * BBWADG scheme on affine triangles (R29-R30), one fused kernel per RK stage.
 *   mesh:  vertices [num_vertices][2], elements [K][3] global vertex ids, counter-clockwise (J > 0;
 *          clockwise triangles are rejected, never reordered); edge f = the edge opposite local vertex f.
 *   c2:    host [K][Mp2] degree-M Bernstein coefficients of c^2, Mp2 = (M+1)(M+2)/2, canonical order
 *          for a2 in 0..M: for a1 in 0..M-a2 (a0 = M - a1 - a2).
 * The context uses the common calls with 3 fields: state Q[K][3][Np2] = (p, u_x, u_y), Np2 =
 * (N+1)(N+2)/2; bbwadg_set_source takes [K][Np2] (the 2D manufactured source of P:646-652);
 * bbwadg_wadg_apply maps [K][Np2] -> [K][Np2].  world_size must be 1. */
typedef struct {
  int64_t num_vertices;
  const double* vertices;   /* [num_vertices][2] */
  int64_t num_elements;
  const int64_t* elements;  /* [num_elements][3] */
} bbwadg_mesh2d;
bbwadg_status bbwadg2d_setup(const bbwadg_mesh2d* mesh, int N, int M, const double* c2_coeffs,
                             const bbwadg_options* opts, bbwadg_ctx* out);

/* ---- in-process partition groups (test/debug: P partitions on one device,
 * halo exchanged by device copies instead of NCCL; validates partitioning,
 * packing, orientation and the interior/boundary split without a cluster) */
bbwadg_status bbwadg_setup_group(const bbwadg_mesh* mesh, int N, int M, const double* c2_coeffs,
                                 const bbwadg_options* opts, int nparts, bbwadg_ctx* out /* [nparts] */);
bbwadg_status bbwadg_group_step(bbwadg_ctx* ctxs, int nparts, double t, double dt);

/* ---- peer-read halo across processes (halo_transport = 1, world_size > 1): CUDA IPC mapping of the
 * partitions' state buffers, so the stage kernel reads neighbour face traces from the owner's Q_in in
 * place (over NVLink between GPUs; also valid for several processes sharing one GPU).
 * bbwadg_ipc_get_handles: out[3][64] = cudaIpcMemHandle_t of this context's two state buffers and of its
 *                         stage-epoch flag (partitioned halo_transport 1 contexts only).
 * bbwadg_ipc_open_peer:   map the handles of rank `peer` (from its bbwadg_ipc_get_handles, exchanged by
 *                         the caller); every rank that owns a neighbour of this partition must be opened.
 * Stages of IPC peers are ordered ON THE DEVICE: before stage e a one-warp kernel waits (acquire, system
 * scope, bounded spin) until every opened peer has published epoch >= e-1, and after the stage the own epoch
 * is published (release), so bbwadg_step / bbwadg_run need no host barrier; a peer that stops advancing
 * makes bbwadg_run fail with BBWADG_ERR_CUDA after ~30 s instead of hanging.  All ranks must call the same
 * sequence of stages (set_state / get_state are not synchronised: barrier around them).
 * bbwadg_stage:           one LSRK45 stage s (0..4) of the state at stage time t + c_s dt (s = 0..4 in order
 *                         is one bbwadg_step); works for every context. */
bbwadg_status bbwadg_ipc_get_handles(bbwadg_ctx ctx, void* out);
bbwadg_status bbwadg_ipc_open_peer(bbwadg_ctx ctx, int peer, const void* handles);
bbwadg_status bbwadg_stage(bbwadg_ctx ctx, int s, double t, double dt);

/* ---- host-only helpers (no GPU needed) */
/* Partition plan of rank `rank` among nparts (the same recursive coordinate bisection and
 * halo ordering bbwadg_setup uses).  sizes[4] = {K_local, n_interior, n_send_faces, n_ghost_faces}.
 * Optional outputs (NULL to skip; call once with NULLs to get the sizes):
 *   gid  [K_local]          global element id of each local element (local order)
 *   send [n_send][4]        (global element, face, destination rank, neighbour global element), message order
 *   recv [n_ghost][4]       (global element, face, source rank, neighbour global element), ghost-slot order */
bbwadg_status bbwadg_partition_plan(const bbwadg_mesh* mesh, int nparts, const int cuts[3], int rank,
                                    int64_t* sizes, int64_t* gid, int64_t* send, int64_t* recv);
/* c_0..c_N of P^{N+M}_N = sum_j c_j E^N_{N-j} (E^N_{N-j})^T (E^{N+M}_N)^T
 * (Thm main / Eq. decomp; Table 1) from the closed-form
 * Bernstein mass eigenvalues (R8). out: N+1 doubles. */
bbwadg_status bbwadg_projection_constants(int N, int M, double* out);
/* c_0..c_N of M^-1 = sum_j c_j E E^T for the reference tetrahedron
 * (Thm bbmass / Eq. mass; Table 2). out: N+1 doubles. */
bbwadg_status bbwadg_mass_inverse_constants(int N, double* out);
/* ncclGetUniqueId into out[128]. */
bbwadg_status bbwadg_nccl_unique_id(void* out);
/* Library build identification string. */
const char* bbwadg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BBWADG_H */
