// extern "C" implementation of include/bbwadg.h.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: named ranges per RK stage / halo (nsys, ncu --nvtx)

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/bbwadg.h"
#include "dispatch.hpp"
#include "mesh.hpp"
#include "nccl_shim.hpp"
#include "elastic_kernel.cuh"
#include "layout2d.hpp"
#include "stage2d_kernel.cuh"
#include "stage_kernel.cuh"
#include "tables.hpp"
#include "layout.hpp"

using namespace bbw;

namespace bbw {
KernelSet get_kernels(int N, int M, int dtype) {
  switch (N) {
    case 1: return get_kernels_N1(M, dtype);
    case 2: return get_kernels_N2(M, dtype);
    case 3: return get_kernels_N3(M, dtype);
    case 4: return get_kernels_N4(M, dtype);
    case 5: return get_kernels_N5(M, dtype);
    case 6: return get_kernels_N6(M, dtype);
    case 7: return get_kernels_N7(M, dtype);
    case 8: return get_kernels_N8(M, dtype);
    case 9: return get_kernels_N9(M, dtype);
    default: return KernelSet();
  }
}
}  // namespace bbw

// Carpenter & Kennedy (1994) 5-stage 2N-storage RK4 (R13)
static const double RK_A[5] = {0.0, -567301805773.0 / 1357537059087.0, -2404267990393.0 / 2016746695238.0,
                               -3550918686646.0 / 2091501179385.0, -1275806237668.0 / 842570457699.0};
static const double RK_B[5] = {1432997174477.0 / 9575080441755.0, 5161836677717.0 / 13612068292357.0,
                               1720146321549.0 / 2090206949498.0, 3134564353537.0 / 4481467310338.0,
                               2277821191437.0 / 14882151754819.0};
static const double RK_C[5] = {0.0, 1432997174477.0 / 9575080441755.0, 2526269341429.0 / 6820363962896.0,
                               2006345519317.0 / 3224310063776.0, 2802321613138.0 / 2924317926251.0};

static thread_local std::string g_last_error;

struct Group;

struct bbwadg_ctx_s {
  int N = 0, M = 0, dtype = 0, device = 0, Np = 0, Mp = 0, Nfp = 0;
  int nfields = 4;       // 4 acoustic (p, u), 9 elastic (v, sigma), 3 for 2D (p, u_x, u_y)
  int dim = 3;           // 2: triangle context (bbwadg2d_setup, NEXT-4)
  bool elastic = false;  // bbwadg_elastic_setup context (NEXT-2)
  size_t rb = 8;  // bytes per real
  double tau_p = 1, tau_u = 1;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int64_t K_global = 0;
  Part part;
  HostTables tables;
  KernelSet ks;
  int grid = 0;
  // device memory
  void* d_tab = nullptr;
  void* d_Q[2] = {nullptr, nullptr};
  int cur = 0;
  void* d_res = nullptr;
  void* d_c2 = nullptr;
  void* d_geo = nullptr;
  int* d_nbr = nullptr;
  uint8_t* d_code = nullptr;
  void* d_src = nullptr;
  void* d_ghost = nullptr;
  void* d_send = nullptr;
  int* d_sendfaces = nullptr;
  int* d_flag = nullptr;
  unsigned int* d_qctr = nullptr;  // stage-kernel work queue: [0] next batch ticket, [1] finished units
  int qch_elastic = 1;             // elastic kernel: unit-batches per ticket (BBWADG_ELASTIC_QCH, A/B knob)
  unsigned long long* d_ptime = nullptr;  // phase timing counters (BBW_PHASE_TIMING builds)
  // peer-read halo (halo_transport 1): owner-rank / owner-local id per ghost slot, and the peers' two
  // state buffers (same-process group members, or CUDA-IPC mappings of other processes)
  int transport = 0;
  int* d_gmap = nullptr;
  void* peer_q[8][2] = {};
  bool peer_ipc[8] = {};
  // device-side stage barrier of IPC peers: own epoch flag (stages completed), the peers' mapped flags
  unsigned long long* d_epoch = nullptr;
  unsigned long long* peer_epoch[8] = {};
  unsigned long long epoch = 0;
  int* d_sync_err = nullptr;
  // multi-GPU
  nccl::Comm comm = nullptr;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
  Group* group = nullptr;
  int group_index = 0;
  // CUDA graphs of one LSRK step (5 stage launches), one per starting state buffer, replayed by bbwadg_run
  cudaStream_t gstream = nullptr;
  cudaEvent_t gev = nullptr;
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};
  double gdt = 0;
  // bookkeeping
  int64_t steps = 0;
  double t = 0;
  std::string err;
};

struct Group {
  std::vector<bbwadg_ctx> parts;
  cudaStream_t stream = nullptr;  // shared by all members, owned by the group
};

namespace {

bbwadg_status fail(bbwadg_ctx c, bbwadg_status s, const std::string& msg) {
  if (c) c->err = msg;
  g_last_error = msg;
  return s;
}

#define CUDA_TRY(ctx, call)                                                                          \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess) {                                                                         \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? BBWADG_ERR_OOM : BBWADG_ERR_CUDA,           \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                               \
    }                                                                                                \
  } while (0)

template <typename R>
void fill_args(bbwadg_ctx c, StageArgs<R>& a) {
  std::memset(&a, 0, sizeof(a));
  a.c2 = static_cast<const R*>(c->d_c2);
  a.geo = static_cast<const R*>(c->d_geo);
  a.nbr = c->d_nbr;
  a.code = c->d_code;
  a.ghost = static_cast<const R*>(c->d_ghost);
  a.src = static_cast<const R*>(c->d_src);
  a.tab = static_cast<const uint8_t*>(c->d_tab);
  a.qctr = c->d_qctr;
  if (c->transport == 1 && c->d_gmap) {
    a.gmap = c->d_gmap;
    for (int r = 0; r < 8; ++r) a.peer[r] = static_cast<const R*>(c->peer_q[r][c->cur]);
  }
  const HostTables& T = c->tables;
  a.tau_p = (R)c->tau_p;
  a.tau_u = (R)c->tau_u;
  for (int j = 0; j < 10; ++j) {
    a.gam[j] = (R)T.gam[j];
    a.lam[j] = (R)T.lam[j];
  }
}

// Elastic stage kernel over local elements [b, e) (Qin/Qout/res: [K][9][Np]).
template <typename R>
bbwadg_status launch_elastic_typed(bbwadg_ctx c, int mode, const void* Qin, void* Qout, int64_t b, int64_t e,
                                   double rk_a, double rk_b, double dt, int grid) {
  ElasticArgs<R> a;
  std::memset(&a, 0, sizeof(a));
  fill_args(c, a.s);
  a.s.Qin = static_cast<const R*>(Qin);
  a.s.Qout = static_cast<R*>(Qout);
  a.s.res = static_cast<R*>(c->d_res);
  a.s.elem_begin = b;
  a.s.elem_end = e;
  a.s.rk_a = (R)rk_a;
  a.s.rk_b = (R)rk_b;
  a.s.dt = (R)dt;
  a.s.mode = mode;
  a.s.qch = c->qch_elastic;
  a.mat = static_cast<const R*>(c->d_c2);
  a.tau_s = (R)c->tau_p;  // elastic contexts: tau_p carries tau_sigma, tau_u carries tau_v (header)
  a.tau_v = (R)c->tau_u;
  cudaError_t err = c->ks.launch_elastic(&a, grid, c->stream);
  if (err != cudaSuccess) return fail(c, BBWADG_ERR_CUDA, std::string("elastic kernel launch: ") + cudaGetErrorString(err));
  return BBWADG_OK;
}

bbwadg_status launch_elastic_pass(bbwadg_ctx c, int mode, const void* Qin, void* Qout, int64_t b, int64_t e,
                                  double rk_a, double rk_b, double dt) {
  const int64_t nb = (e - b + c->ks.elastic_elems_per_cta - 1) / c->ks.elastic_elems_per_cta;
  const int grid = (int)std::min<int64_t>(nb, c->grid);
  return c->dtype == BBWADG_F64 ? launch_elastic_typed<double>(c, mode, Qin, Qout, b, e, rk_a, rk_b, dt, grid)
                                : launch_elastic_typed<float>(c, mode, Qin, Qout, b, e, rk_a, rk_b, dt, grid);
}

// 2D (triangle) stage kernel over local elements [b, e) (Q: [K][3][Np2]).
template <typename R>
bbwadg_status launch_2d_typed(bbwadg_ctx c, int mode, const void* Qin, void* Qout, int64_t b, int64_t e, double rk_a,
                              double rk_b, double dt, double tstage, int grid) {
  Stage2DArgs<R> a;
  std::memset(&a, 0, sizeof(a));
  a.Qin = static_cast<const R*>(Qin);
  a.Qout = static_cast<R*>(Qout);
  a.res = static_cast<R*>(c->d_res);
  a.c2 = static_cast<const R*>(c->d_c2);
  a.geo = static_cast<const R*>(c->d_geo);
  a.nbr = c->d_nbr;
  a.code = c->d_code;
  a.src = static_cast<const R*>(c->d_src);
  a.tab = static_cast<const uint8_t*>(c->d_tab);
  a.elem_begin = b;
  a.elem_end = e;
  a.rk_a = (R)rk_a;
  a.rk_b = (R)rk_b;
  a.dt = (R)dt;
  a.src_amp = (R)std::sin(M_PI * tstage);
  a.tau_p = (R)c->tau_p;
  a.tau_u = (R)c->tau_u;
  for (int j = 0; j < 10; ++j) a.gam[j] = (R)c->tables.gam[j];
  a.mode = mode;
  cudaError_t err = c->ks.launch_stage(&a, grid, c->stream);
  if (err != cudaSuccess) return fail(c, BBWADG_ERR_CUDA, std::string("2D kernel launch: ") + cudaGetErrorString(err));
  return BBWADG_OK;
}

bbwadg_status launch_2d_pass(bbwadg_ctx c, int mode, const void* Qin, void* Qout, int64_t b, int64_t e, double rk_a,
                             double rk_b, double dt, double tstage) {
  const int64_t nb = (e - b + c->ks.elems_per_cta - 1) / c->ks.elems_per_cta;
  const int grid = (int)std::min<int64_t>(nb, c->grid);
  return c->dtype == BBWADG_F64 ? launch_2d_typed<double>(c, mode, Qin, Qout, b, e, rk_a, rk_b, dt, tstage, grid)
                                : launch_2d_typed<float>(c, mode, Qin, Qout, b, e, rk_a, rk_b, dt, tstage, grid);
}

// Launch one kernel pass over local elements [b, e).
bbwadg_status launch_pass(bbwadg_ctx c, int mode, const void* Qin, void* Qout, int64_t b, int64_t e, double rk_a,
                          double rk_b, double dt, double tstage, int grid_cap = 0) {
  if (e <= b) return BBWADG_OK;
  if (c->elastic) return launch_elastic_pass(c, mode, Qin, Qout, b, e, rk_a, rk_b, dt);
  if (c->dim == 2) return launch_2d_pass(c, mode, Qin, Qout, b, e, rk_a, rk_b, dt, tstage);
  int64_t nb = (e - b + c->ks.elems_per_cta - 1) / c->ks.elems_per_cta;
  int grid = (int)std::min<int64_t>(nb, grid_cap > 0 ? grid_cap : c->grid);
  // work-queue ticket size: one unit-batch when every CTA slot runs >= 1000 batches (SM drift would otherwise
  // spread the in-flight window; config 5: +1.7 % over 2), two below (amortises the atomic; +3.8 % at (5,3) on
  // 1.57M elements).  A/B: profiles/r2s3_workqueue_ab.txt
  const int qch = nb >= 1000 * (int64_t)grid ? 1 : 2;
  cudaError_t err;
  if (c->dtype == BBWADG_F64) {
    StageArgs<double> a;
    fill_args(c, a);
    a.Qin = static_cast<const double*>(Qin);
    a.Qout = static_cast<double*>(Qout);
    a.res = static_cast<double*>(c->d_res);
    a.elem_begin = b;
    a.elem_end = e;
    a.rk_a = rk_a;
    a.rk_b = rk_b;
    a.dt = dt;
    a.src_amp = std::sin(M_PI * tstage);
    a.mode = mode;
    a.ptime = c->d_ptime;
    a.qch = qch;
    err = c->ks.launch_stage(&a, grid, c->stream);
  } else {
    StageArgs<float> a;
    fill_args(c, a);
    a.Qin = static_cast<const float*>(Qin);
    a.Qout = static_cast<float*>(Qout);
    a.res = static_cast<float*>(c->d_res);
    a.elem_begin = b;
    a.elem_end = e;
    a.rk_a = (float)rk_a;
    a.rk_b = (float)rk_b;
    a.dt = (float)dt;
    a.src_amp = (float)std::sin(M_PI * tstage);
    a.mode = mode;
    a.ptime = c->d_ptime;
    a.qch = qch;
    err = c->ks.launch_stage(&a, grid, c->stream);
  }
  if (err != cudaSuccess) return fail(c, BBWADG_ERR_CUDA, std::string("stage kernel launch: ") + cudaGetErrorString(err));
  return BBWADG_OK;
}

const uint16_t* fnode_ptr(bbwadg_ctx c) {
  const TabLayout L = tab_layout(c->N, c->M, (int)c->rb);
  return reinterpret_cast<const uint16_t*>(static_cast<const uint8_t*>(c->d_tab) + L.fnode);
}

struct NvtxRange {  // RAII NVTX range (no-op without a tool attached)
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// NCCL halo for source state Q: pack on the comm stream, grouped send/recv, event.
bbwadg_status halo_nccl(bbwadg_ctx c, const void* Q) {
  NvtxRange range("bbwadg halo (pack + NCCL send/recv)");
  const Part& P = c->part;
  const int64_t nsend = P.send_off.back();
  CUDA_TRY(c, cudaEventRecord(c->ev_ready, c->stream));
  CUDA_TRY(c, cudaStreamWaitEvent(c->comm_stream, c->ev_ready, 0));
  CUDA_TRY(c, c->ks.launch_pack(Q, c->d_geo, c->d_sendfaces, (int)nsend, fnode_ptr(c), c->d_send, c->comm_stream));
  const size_t per_face = 2 * (size_t)c->Nfp;  // p and u.n per face node (Eq. sdf needs only [[p]], n.[[u]])
  int dt = c->dtype == BBWADG_F64 ? nccl::kDouble : nccl::kFloat;
  if (nccl::group_start() != 0) return fail(c, BBWADG_ERR_NCCL, "ncclGroupStart failed");
  for (int r = 0; r < P.nparts; ++r) {
    int64_t ns = P.send_off[r + 1] - P.send_off[r];
    int64_t nr = P.recv_off[r + 1] - P.recv_off[r];
    if (ns > 0) {
      const char* sp = static_cast<const char*>(c->d_send) + P.send_off[r] * per_face * c->rb;
      if (nccl::send(sp, ns * per_face, dt, r, c->comm, c->comm_stream) != 0)
        return fail(c, BBWADG_ERR_NCCL, "ncclSend failed");
    }
    if (nr > 0) {
      char* rp = static_cast<char*>(c->d_ghost) + P.recv_off[r] * per_face * c->rb;
      if (nccl::recv(rp, nr * per_face, dt, r, c->comm, c->comm_stream) != 0)
        return fail(c, BBWADG_ERR_NCCL, "ncclRecv failed");
    }
  }
  if (nccl::group_end() != 0) return fail(c, BBWADG_ERR_NCCL, std::string("ncclGroupEnd failed: ") + nccl::last_error(c->comm));
  CUDA_TRY(c, cudaEventRecord(c->ev_halo, c->comm_stream));
  return BBWADG_OK;
}

// Device-side barrier between LSRK stages of IPC peers (peer-read halo): before stage e every peer must have
// completed stage e-1 (its stage output is this stage's neighbour input, and it no longer reads the buffer
// this stage overwrites).  One thread per peer polls the peer's epoch flag (acquire, system scope) with a
// bounded spin (timeout -> error flag, no hang); after the stage one thread publishes the own epoch (release).
struct PeerFlags {
  const unsigned long long* f[8];
  int n;
};
__global__ void peer_wait_kernel(PeerFlags pf, unsigned long long target, int* err) {
  const int i = threadIdx.x;
  if (i >= pf.n) return;
  const long long t0 = clock64();
  for (;;) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(pf.f[i]) : "memory");
    if (v >= target) break;
    if (clock64() - t0 > 60000000000LL) {  // ~30 s at 2 GHz
      atomicExch(err, 1);
      break;
    }
    __nanosleep(2000);
  }
}
__global__ void epoch_signal_kernel(unsigned long long* flag, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(v) : "memory");
}

// One pass (stage or rhs) over all local elements including the halo exchange when partitioned.
bbwadg_status full_pass(bbwadg_ctx c, int mode, const void* Qin, void* Qout, double rk_a, double rk_b, double dt,
                        double tstage) {
  static const char* kNames[3] = {"bbwadg stage (LSRK)", "bbwadg rhs", "bbwadg wadg_apply"};
  NvtxRange range(kNames[mode < 0 || mode > 2 ? 0 : mode]);
  const Part& P = c->part;
  if (P.nparts > 1 && c->transport == 1) {
    // peer reads: the boundary elements read the owners' Q_in in place (the caller guarantees the peers
    // finished writing it: same stream for groups, a barrier between stages across processes)
    for (int r = 0; r < P.nparts; ++r)
      if (r != P.rank && P.recv_off[r + 1] > P.recv_off[r] && !c->peer_q[r][c->cur])
        return fail(c, BBWADG_ERR_INVALID_ARG, "peer-read halo: a neighbour partition's state is not mapped");
    if (Qin != c->d_Q[c->cur]) return fail(c, BBWADG_ERR_INVALID_ARG, "peer-read halo works on the context state only");
    PeerFlags pf{};
    for (int r = 0; r < P.nparts && r < 8; ++r)
      if (c->peer_epoch[r]) pf.f[pf.n++] = c->peer_epoch[r];
    if (pf.n > 0) {
      peer_wait_kernel<<<1, 32, 0, c->stream>>>(pf, c->epoch, c->d_sync_err);
      CUDA_TRY(c, cudaGetLastError());
    }
    bbwadg_status st = launch_pass(c, mode, Qin, Qout, 0, P.K_local, rk_a, rk_b, dt, tstage);
    if (st) return st;
    if (c->d_epoch) {
      epoch_signal_kernel<<<1, 1, 0, c->stream>>>(c->d_epoch, ++c->epoch);
      CUDA_TRY(c, cudaGetLastError());
    }
    return BBWADG_OK;
  }
  if (P.nparts > 1 && c->comm) {
    bbwadg_status s = halo_nccl(c, Qin);
    if (s) return s;
    // the persistent interior pass leaves two SMs' worth of CTAs free, so the pack and NCCL kernels on
    // the comm stream run concurrently with it (full occupancy would hold them back until it drains)
    const int cap = std::max(c->ks.blocks_per_sm(), c->grid - 2 * c->ks.blocks_per_sm());
    s = launch_pass(c, mode, Qin, Qout, 0, P.n_interior, rk_a, rk_b, dt, tstage, cap);
    if (s) return s;
    CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_halo, 0));
    return launch_pass(c, mode, Qin, Qout, P.n_interior, P.K_local, rk_a, rk_b, dt, tstage);
  }
  return launch_pass(c, mode, Qin, Qout, 0, P.K_local, rk_a, rk_b, dt, tstage);
}

size_t state_bytes(bbwadg_ctx c) { return (size_t)c->part.K_local * c->nfields * c->Np * c->rb; }

template <typename R>
__global__ void nonfinite_kernel(const R* __restrict__ q, long long n, int* flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (!isfinite(q[i])) {
      *flag = 1;
      return;
    }
}

bbwadg_status upload_real(bbwadg_ctx c, void** dst, const std::vector<double>& host) {
  size_t n = host.size();
  if (n == 0) {
    *dst = nullptr;
    return BBWADG_OK;
  }
  CUDA_TRY(c, cudaMalloc(dst, n * c->rb));
  if (c->dtype == BBWADG_F64) {
    CUDA_TRY(c, cudaMemcpy(*dst, host.data(), n * 8, cudaMemcpyHostToDevice));
  } else {
    std::vector<float> f(host.begin(), host.end());
    CUDA_TRY(c, cudaMemcpy(*dst, f.data(), n * 4, cudaMemcpyHostToDevice));
  }
  return BBWADG_OK;
}

// c^2_M positivity check (R16): values at the degree-(M+2) barycentric lattice of
// each element (includes the 4 vertices); basis values precomputed once.
struct C2Checker {
  int M = 0, npts = 0, mp = 0;
  std::vector<double> B;  // [npts][mp]
  explicit C2Checker(int M_) : M(M_) {
    int q = M + 2;
    auto idx = indices3(M);
    mp = (int)idx.size();
    for (int b3 = 0; b3 <= q; ++b3)
      for (int b2 = 0; b2 <= q - b3; ++b2)
        for (int b1 = 0; b1 <= q - b3 - b2; ++b1) {
          long double lam[4] = {(long double)(q - b1 - b2 - b3) / q, (long double)b1 / q, (long double)b2 / q,
                                (long double)b3 / q};
          for (int i = 0; i < mp; ++i) {
            long double mult = 1, term = 1;
            for (int m = 2; m <= M; ++m) mult *= m;
            for (int j = 0; j < 4; ++j) {
              for (int m = 2; m <= idx[i].a[j]; ++m) mult /= m;
              for (int p = 0; p < idx[i].a[j]; ++p) term *= lam[j];
            }
            B.push_back((double)(mult * term));
          }
          ++npts;
        }
  }
  // returns the minimum sampled value
  double min_value(const double* c) const {
    double mn = 1e300;
    for (int p = 0; p < npts; ++p) {
      double v = 0;
      for (int i = 0; i < mp; ++i) v += B[(size_t)p * mp + i] * c[i];
      mn = v < mn ? v : mn;
    }
    return mn;
  }
};

// c2: acoustic [rows][Mp] c^2_M; elastic (elastic = true) [K][3][Mp] (rho^-1, lambda, mu) interleaved per element
bbwadg_status setup_one(const GlobalMesh& g, int N, int M, const double* c2, const bbwadg_options& o, int rank,
                        int nparts, cudaStream_t shared_stream, bbwadg_ctx* out, bool elastic = false) {
  std::unique_ptr<bbwadg_ctx_s> c(new bbwadg_ctx_s());
  struct Cleanup {  // release device resources on every early-error return
    std::unique_ptr<bbwadg_ctx_s>& p;
    ~Cleanup() {
      if (p) bbwadg_destroy(p.release());
    }
  } cleanup{c};
  c->N = N;
  c->M = M;
  c->dtype = o.dtype;
  c->device = o.device;
  c->rb = o.dtype == BBWADG_F64 ? 8 : 4;
  c->tau_p = o.tau_p;
  c->tau_u = o.tau_u;
  c->Np = np3(N);
  c->Mp = np3(M);
  c->Nfp = np2(N);
  c->K_global = g.K;
  c->elastic = elastic;
  c->nfields = elastic ? 9 : 4;
  CUDA_TRY(c.get(), cudaSetDevice(o.device));
  c->ks = get_kernels(N, M, o.dtype);
  if (!c->ks.launch_stage || (elastic && !c->ks.launch_elastic))
    return fail(nullptr, BBWADG_ERR_UNSUPPORTED, "no kernel instantiation for this (N, M, dtype)");
  CUDA_TRY(c.get(), c->ks.prepare());
  if (elastic) CUDA_TRY(c.get(), c->ks.prepare_elastic());
  int nsm = 0;
  CUDA_TRY(c.get(), cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, o.device));
  c->grid = nsm * (elastic ? c->ks.elastic_blocks_per_sm() : c->ks.blocks_per_sm());
  if (const char* e = getenv("BBWADG_BLOCKS_PER_SM")) {  // tuning: occupancy sensitivity experiments
    const int b = atoi(e);
    if (b > 0 && b < c->ks.blocks_per_sm()) c->grid = nsm * b;
  }
  // elastic work-queue ticket size: 1 measured best at (7,2) (2.08 vs 2.03 / 2.00e10 for 2 / 4; (5,1), (9,2) within
  // 0.7 %); BBWADG_ELASTIC_QCH overrides (A/B knob)
  if (const char* e = getenv("BBWADG_ELASTIC_QCH")) c->qch_elastic = std::max(1, atoi(e));
  if (const char* e = getenv("BBWADG_FORCE_BLOCKS_PER_SM")) {  // tuning: override the occupancy query (TMEM study)
    const int b = atoi(e);
    if (b > 0) c->grid = nsm * b;
  }
  // NULL selects the legacy default stream (stream 0), so that work is ordered with
  // torch's default stream and every other legacy-stream user (cuBLAS convention).
  c->stream = shared_stream ? shared_stream : static_cast<cudaStream_t>(o.cuda_stream);
  c->own_stream = false;
  c->part = build_part(g, rank, nparts);
  const Part& P = c->part;
  // tables
  try {
    c->tables = build_tables(N, M, (int)c->rb);
  } catch (const std::exception& e) {
    return fail(nullptr, BBWADG_ERR_UNSUPPORTED, e.what());
  }
  CUDA_TRY(c.get(), cudaMalloc(&c->d_tab, c->tables.blob.size()));
  CUDA_TRY(c.get(), cudaMemcpy(c->d_tab, c->tables.blob.data(), c->tables.blob.size(), cudaMemcpyHostToDevice));
  // per-element inputs in local order
  const int64_t KL = P.K_local;
  const int W = elastic ? 3 * c->Mp : c->Mp;  // material reals per element
  std::vector<double> geo(12 * KL), c2l((size_t)KL * W);
  // c^2 rows: global order, or only the listed global ids (o.c2_gids, sorted lookup)
  std::vector<std::pair<int64_t, int64_t>> c2map;
  if (o.c2_gids) {
    c2map.resize(o.c2_rows);
    for (int64_t r = 0; r < o.c2_rows; ++r) c2map[r] = {o.c2_gids[r], r};
    std::sort(c2map.begin(), c2map.end());
  }
  std::vector<int64_t> c2row(KL);
  for (int64_t i = 0; i < KL; ++i) {
    if (!o.c2_gids) {
      c2row[i] = P.gid[i];
      continue;
    }
    auto it = std::lower_bound(c2map.begin(), c2map.end(), std::make_pair(P.gid[i], (int64_t)-1));
    if (it == c2map.end() || it->first != P.gid[i]) {
      std::ostringstream os;
      os << "c2_gids lacks global element " << P.gid[i] << " owned by rank " << rank;
      return fail(nullptr, BBWADG_ERR_INVALID_ARG, os.str());
    }
    c2row[i] = it->second;
  }
  C2Checker chk(M);
  int64_t bad = -1;
  double badv = 0;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < KL; ++i) {
    element_gradients(g, P.gid[i], &geo[12 * i]);
    const double* ci = c2 + (size_t)c2row[i] * W;
    std::memcpy(&c2l[(size_t)i * W], ci, sizeof(double) * W);
    if (o.check_c2 && elastic) {
      // rho^-1 > 0, lambda + 2 mu > 0 (P-wave modulus), mu >= 0 at the sample points (R25; mu = 0 is the
      // acoustic limit)
      std::vector<double> pm(c->Mp);
      for (int b = 0; b < c->Mp; ++b) pm[b] = ci[c->Mp + b] + 2.0 * ci[2 * c->Mp + b];
      const double m0 = chk.min_value(ci), m1 = chk.min_value(pm.data()), m2 = chk.min_value(ci + 2 * c->Mp);
      if (!(m0 > 0) || !(m1 > 0) || !(m2 >= 0)) {
#pragma omp critical
        {
          if (bad < 0 || P.gid[i] < bad) {
            bad = P.gid[i];
            badv = std::min(m0, std::min(m1, m2));
          }
        }
      }
    } else if (o.check_c2) {
      // convex hull property: all Bernstein coefficients > 0 => c^2_M > 0 on the element
      bool allpos = true;
      for (int b = 0; b < c->Mp; ++b) allpos = allpos && (ci[b] > 0);
      double mn = allpos ? 1.0 : chk.min_value(ci);
      if (!(mn > 0)) {
#pragma omp critical
        {
          if (bad < 0 || P.gid[i] < bad) {
            bad = P.gid[i];
            badv = mn;
          }
        }
      }
    }
  }
  if (bad >= 0) {
    std::ostringstream os;
    os << (elastic ? "rho^-1 / lambda + 2 mu / mu" : "c^2_M") << " is not positive in element " << bad
       << " (sampled value " << badv << ")";
    return fail(nullptr, BBWADG_ERR_NONPOSITIVE_C2, os.str());
  }
  bbwadg_status s;
  if ((s = upload_real(c.get(), &c->d_geo, geo))) return fail(nullptr, s, c->err);
  if ((s = upload_real(c.get(), &c->d_c2, c2l))) return fail(nullptr, s, c->err);
  CUDA_TRY(c.get(), cudaMalloc(&c->d_nbr, sizeof(int) * 4 * std::max<int64_t>(KL, 1)));
  CUDA_TRY(c.get(), cudaMemcpy(c->d_nbr, P.nbr.data(), sizeof(int) * 4 * KL, cudaMemcpyHostToDevice));
  CUDA_TRY(c.get(), cudaMalloc(&c->d_code, 4 * std::max<int64_t>(KL, 1)));
  CUDA_TRY(c.get(), cudaMemcpy(c->d_code, P.code.data(), 4 * KL, cudaMemcpyHostToDevice));
  const size_t sb = state_bytes(c.get());
  for (int b = 0; b < 2; ++b) {
    CUDA_TRY(c.get(), cudaMalloc(&c->d_Q[b], std::max<size_t>(sb, 16)));
    CUDA_TRY(c.get(), cudaMemset(c->d_Q[b], 0, sb));
  }
  CUDA_TRY(c.get(), cudaMalloc(&c->d_res, std::max<size_t>(sb, 16)));
  CUDA_TRY(c.get(), cudaMemset(c->d_res, 0, sb));
  CUDA_TRY(c.get(), cudaMalloc(&c->d_flag, sizeof(int)));
  CUDA_TRY(c.get(), cudaMalloc(&c->d_qctr, 2 * sizeof(unsigned int)));  // zero between launches (self-reset)
  CUDA_TRY(c.get(), cudaMemset(c->d_qctr, 0, 2 * sizeof(unsigned int)));
  if (getenv("BBWADG_PHASE_TIMING")) {
    CUDA_TRY(c.get(), cudaMalloc(&c->d_ptime, 32 * sizeof(unsigned long long)));
    CUDA_TRY(c.get(), cudaMemset(c->d_ptime, 0, 32 * sizeof(unsigned long long)));
  }
  const int64_t nghost = P.num_ghost(), nsend = P.send_off.empty() ? 0 : P.send_off.back();
  c->transport = o.halo_transport;
  if (c->transport == 1 && nparts > 1) {
    CUDA_TRY(c.get(), cudaMalloc(&c->d_epoch, 256));  // own allocation: exported by CUDA IPC
    CUDA_TRY(c.get(), cudaMemset(c->d_epoch, 0, 256));
  }
  if (c->transport == 1 && nghost > 0) {
    CUDA_TRY(c.get(), cudaMalloc(&c->d_gmap, sizeof(int) * 2 * nghost));
    CUDA_TRY(c.get(), cudaMemcpy(c->d_gmap, P.gmap.data(), sizeof(int) * 2 * nghost, cudaMemcpyHostToDevice));
  }
  const size_t per_face = 2 * (size_t)c->Nfp * c->rb;  // halo: p and u.n per face node
  if (nghost > 0) CUDA_TRY(c.get(), cudaMalloc(&c->d_ghost, nghost * per_face));
  if (nsend > 0) {
    CUDA_TRY(c.get(), cudaMalloc(&c->d_send, nsend * per_face));
    CUDA_TRY(c.get(), cudaMalloc(&c->d_sendfaces, sizeof(int) * 2 * nsend));
    CUDA_TRY(c.get(), cudaMemcpy(c->d_sendfaces, P.send_faces.data(), sizeof(int) * 2 * nsend, cudaMemcpyHostToDevice));
  }
  CUDA_TRY(c.get(), cudaDeviceSynchronize());
  *out = c.release();
  return BBWADG_OK;
}

bbwadg_status prepare_global(const bbwadg_mesh* mesh, int N, int M, const double* c2, const bbwadg_options* opts,
                             int nparts, GlobalMesh& g) {
  if (!mesh || !mesh->vertices || !mesh->elements || mesh->num_elements < 1 || mesh->num_vertices < 4 || !c2)
    return fail(nullptr, BBWADG_ERR_INVALID_ARG, "mesh/c2 pointers or sizes invalid");
  if (N < 1 || N > BBWADG_MAX_N || M < 0 || M > N)
    return fail(nullptr, BBWADG_ERR_UNSUPPORTED, "need 1 <= N <= 9 and 0 <= M <= N");
  if (opts && opts->dtype != BBWADG_F64 && opts->dtype != BBWADG_F32)
    return fail(nullptr, BBWADG_ERR_UNSUPPORTED, "dtype must be BBWADG_F64 or BBWADG_F32");
  if (opts && (opts->tau_p < 0 || opts->tau_u < 0)) return fail(nullptr, BBWADG_ERR_INVALID_ARG, "tau must be >= 0");
  if (opts && (opts->halo_transport < 0 || opts->halo_transport > 1))
    return fail(nullptr, BBWADG_ERR_INVALID_ARG, "halo_transport must be 0 (pack + NCCL) or 1 (peer reads)");
  if (opts && opts->halo_transport == 1 && nparts > 8)
    return fail(nullptr, BBWADG_ERR_UNSUPPORTED, "peer-read halo supports up to 8 partitions (one NVLink domain)");
  g.K = mesh->num_elements;
  g.nv = mesh->num_vertices;
  g.V = mesh->vertices;
  g.EV = mesh->elements;
  std::string e = check_orientation(g);
  if (!e.empty()) return fail(nullptr, BBWADG_ERR_MESH, e);
  e = build_connectivity(g);
  if (!e.empty()) return fail(nullptr, BBWADG_ERR_MESH, e);
  e = partition(g, nparts, opts ? opts->partition : nullptr);
  if (!e.empty()) return fail(nullptr, BBWADG_ERR_INVALID_ARG, e);
  return BBWADG_OK;
}

}  // namespace

extern "C" {

void bbwadg_default_options(bbwadg_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->dtype = BBWADG_F64;
  o->tau_p = 1.0;
  o->tau_u = 1.0;
  o->world_size = 1;
  o->check_c2 = 1;
}

bbwadg_status bbwadg_setup(const bbwadg_mesh* mesh, int N, int M, const double* c2_coeffs, const bbwadg_options* opts,
                           bbwadg_ctx* out) {
  if (!out) return fail(nullptr, BBWADG_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  bbwadg_options o;
  bbwadg_default_options(&o);
  if (opts) o = *opts;
  if (o.world_size < 1 || o.rank < 0 || o.rank >= o.world_size)
    return fail(nullptr, BBWADG_ERR_INVALID_ARG, "rank/world_size invalid");
  if (o.world_size > 1 && o.halo_transport == 0 && !o.nccl_unique_id)
    return fail(nullptr, BBWADG_ERR_INVALID_ARG, "world_size > 1 needs nccl_unique_id (halo_transport 0)");
  // argument and mesh validation first (host only), then the device
  GlobalMesh g;
  bbwadg_status s = prepare_global(mesh, N, M, c2_coeffs, &o, o.world_size, g);
  if (s) return s;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) return fail(nullptr, BBWADG_ERR_NO_DEVICE, "no CUDA device");
  s = setup_one(g, N, M, c2_coeffs, o, o.rank, o.world_size, nullptr, out);
  if (s) return s;
  bbwadg_ctx c = *out;
  if (o.world_size > 1 && o.halo_transport == 0) {
    std::string why;
    if (!nccl::load(why)) {
      bbwadg_destroy(c);
      *out = nullptr;
      return fail(nullptr, BBWADG_ERR_NCCL, why);
    }
    if (nccl::comm_init_rank(&c->comm, o.world_size, o.nccl_unique_id, o.rank) != 0) {
      bbwadg_destroy(c);
      *out = nullptr;
      return fail(nullptr, BBWADG_ERR_NCCL, "ncclCommInitRank failed");
    }
    cudaError_t ce = cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking);
    if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming);
    if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming);
    if (ce != cudaSuccess) {  // never hand out a half-built context
      bbwadg_destroy(c);
      *out = nullptr;
      return fail(nullptr, BBWADG_ERR_CUDA, std::string("comm stream/events: ") + cudaGetErrorString(ce));
    }
  }
  return BBWADG_OK;
}

bbwadg_status bbwadg_elastic_setup(const bbwadg_mesh* mesh, int N, int M, const double* rho_inv,
                                   const double* lambda, const double* mu, const bbwadg_options* opts,
                                   bbwadg_ctx* out) {
  if (!out) return fail(nullptr, BBWADG_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (!rho_inv || !lambda || !mu) return fail(nullptr, BBWADG_ERR_INVALID_ARG, "material pointers must not be NULL");
  bbwadg_options o;
  bbwadg_default_options(&o);
  if (opts) o = *opts;
  if (o.world_size != 1 || o.rank != 0)
    return fail(nullptr, BBWADG_ERR_UNSUPPORTED, "elastic contexts run on one GPU (world_size 1)");
  if (o.c2_gids) return fail(nullptr, BBWADG_ERR_INVALID_ARG, "c2_gids is not used by elastic contexts");
  GlobalMesh g;
  bbwadg_status s = prepare_global(mesh, N, M, rho_inv, &o, 1, g);
  if (s) return s;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) return fail(nullptr, BBWADG_ERR_NO_DEVICE, "no CUDA device");
  const int Mp = np3(M);
  std::vector<double> mat((size_t)g.K * 3 * Mp);
  for (int64_t k = 0; k < g.K; ++k) {
    std::memcpy(&mat[(size_t)k * 3 * Mp], rho_inv + (size_t)k * Mp, sizeof(double) * Mp);
    std::memcpy(&mat[(size_t)k * 3 * Mp + Mp], lambda + (size_t)k * Mp, sizeof(double) * Mp);
    std::memcpy(&mat[(size_t)k * 3 * Mp + 2 * Mp], mu + (size_t)k * Mp, sizeof(double) * Mp);
  }
  return setup_one(g, N, M, mat.data(), o, 0, 1, nullptr, out, true);
}

bbwadg_status bbwadg2d_setup(const bbwadg_mesh2d* mesh, int N, int M, const double* c2, const bbwadg_options* opts,
                             bbwadg_ctx* out) {
  if (!out) return fail(nullptr, BBWADG_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  bbwadg_options o;
  bbwadg_default_options(&o);
  if (opts) o = *opts;
  if (!mesh || !mesh->vertices || !mesh->elements || mesh->num_elements < 1 || mesh->num_vertices < 3 || !c2)
    return fail(nullptr, BBWADG_ERR_INVALID_ARG, "mesh/c2 pointers or sizes invalid");
  if (N < 1 || N > BBWADG_MAX_N || M < 0 || M > N)
    return fail(nullptr, BBWADG_ERR_UNSUPPORTED, "need 1 <= N <= 9 and 0 <= M <= N");
  if (o.dtype != BBWADG_F64 && o.dtype != BBWADG_F32)
    return fail(nullptr, BBWADG_ERR_UNSUPPORTED, "dtype must be BBWADG_F64 or BBWADG_F32");
  if (o.tau_p < 0 || o.tau_u < 0) return fail(nullptr, BBWADG_ERR_INVALID_ARG, "tau must be >= 0");
  if (o.world_size != 1 || o.rank != 0 || o.c2_gids)
    return fail(nullptr, BBWADG_ERR_UNSUPPORTED, "2D contexts run on one GPU (world_size 1, no c2_gids)");
  const int64_t K = mesh->num_elements, nv = mesh->num_vertices;
  const double* V = mesh->vertices;
  const int64_t* E = mesh->elements;
  // host mesh processing: orientation, edge connectivity by global vertex pairs, gradients, codes
  static const int EV[3][2] = {{1, 2}, {0, 2}, {0, 1}};
  std::vector<double> geo(6 * K);
  std::vector<int32_t> nbr(3 * K, -1);
  std::vector<uint8_t> code(3 * K, 0);
  std::vector<std::pair<std::pair<int64_t, int64_t>, int64_t>> keys;  // ((min, max), 3 k + f)
  keys.reserve(3 * K);
  for (int64_t k = 0; k < K; ++k) {
    int64_t g[3];
    for (int i = 0; i < 3; ++i) {
      g[i] = E[3 * k + i];
      if (g[i] < 0 || g[i] >= nv) return fail(nullptr, BBWADG_ERR_MESH, "vertex id out of range");
    }
    const double ax = V[2 * g[1]] - V[2 * g[0]], ay = V[2 * g[1] + 1] - V[2 * g[0] + 1];
    const double bx = V[2 * g[2]] - V[2 * g[0]], by = V[2 * g[2] + 1] - V[2 * g[0] + 1];
    const double det = ax * by - ay * bx;
    if (!(det > 0)) {
      std::ostringstream os;
      os << "triangle " << k << " is not positively oriented (det " << det << ")";
      return fail(nullptr, BBWADG_ERR_MESH, os.str());
    }
    // l1, l2 = inverse of [a b]; grad l0 = -(grad l1 + grad l2)
    const double g1x = by / det, g1y = -bx / det, g2x = -ay / det, g2y = ax / det;
    double* gg = &geo[6 * k];
    gg[0] = -(g1x + g2x);
    gg[1] = -(g1y + g2y);
    gg[2] = g1x;
    gg[3] = g1y;
    gg[4] = g2x;
    gg[5] = g2y;
    for (int f = 0; f < 3; ++f) {
      const int64_t u = g[EV[f][0]], w = g[EV[f][1]];
      keys.push_back({{std::min(u, w), std::max(u, w)}, 3 * k + f});
    }
  }
  std::sort(keys.begin(), keys.end());
  for (size_t i = 0; i < keys.size();) {
    size_t j = i;
    while (j < keys.size() && keys[j].first == keys[i].first) ++j;
    if (j - i > 2) return fail(nullptr, BBWADG_ERR_MESH, "edge shared by more than two triangles");
    if (j - i == 2) {
      const int64_t s0 = keys[i].second, s1 = keys[i + 1].second;
      const int64_t k0 = s0 / 3, k1 = s1 / 3;
      const int f0 = (int)(s0 % 3), f1 = (int)(s1 % 3);
      const int flip = E[3 * k0 + EV[f0][0]] != E[3 * k1 + EV[f1][0]];  // edges run opposite ways
      nbr[3 * k0 + f0] = (int32_t)k1;
      nbr[3 * k1 + f1] = (int32_t)k0;
      code[3 * k0 + f0] = (uint8_t)(2 * f1 + flip);
      code[3 * k1 + f1] = (uint8_t)(2 * f0 + flip);
    }
    i = j;
  }
  // c^2_M > 0: coefficients positive (convex hull), else sampled on the degree-(M+2) lattice
  const int Mp = (M + 1) * (M + 2) / 2;
  if (o.check_c2) {
    const int qd = M + 2;
    for (int64_t k = 0; k < K; ++k) {
      const double* ck = c2 + (size_t)k * Mp;
      bool allpos = true;
      for (int b = 0; b < Mp; ++b) allpos = allpos && ck[b] > 0;
      if (allpos) continue;
      for (int p2 = 0; p2 <= qd; ++p2)
        for (int p1 = 0; p1 <= qd - p2; ++p1) {
          const double l[3] = {(double)(qd - p1 - p2) / qd, (double)p1 / qd, (double)p2 / qd};
          double v = 0;
          int bi = 0;
          for (int b2 = 0; b2 <= M; ++b2)
            for (int b1 = 0; b1 <= M - b2; ++b1, ++bi) {
              const int b0 = M - b1 - b2;
              double mult = 1;
              for (int t = 2; t <= M; ++t) mult *= t;
              for (int t = 2; t <= b0; ++t) mult /= t;
              for (int t = 2; t <= b1; ++t) mult /= t;
              for (int t = 2; t <= b2; ++t) mult /= t;
              v += ck[bi] * mult * std::pow(l[0], b0) * std::pow(l[1], b1) * std::pow(l[2], b2);
            }
          if (!(v > 0)) {
            std::ostringstream os;
            os << "c^2_M is not positive in element " << k << " (sampled value " << v << ")";
            return fail(nullptr, BBWADG_ERR_NONPOSITIVE_C2, os.str());
          }
        }
    }
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) return fail(nullptr, BBWADG_ERR_NO_DEVICE, "no CUDA device");
  std::unique_ptr<bbwadg_ctx_s> c(new bbwadg_ctx_s());
  struct Cleanup {
    std::unique_ptr<bbwadg_ctx_s>& p;
    ~Cleanup() {
      if (p) bbwadg_destroy(p.release());
    }
  } cleanup{c};
  c->N = N;
  c->M = M;
  c->dim = 2;
  c->nfields = 3;
  c->dtype = o.dtype;
  c->device = o.device;
  c->rb = o.dtype == BBWADG_F64 ? 8 : 4;
  c->tau_p = o.tau_p;
  c->tau_u = o.tau_u;
  c->Np = (N + 1) * (N + 2) / 2;
  c->Mp = Mp;
  c->Nfp = N + 1;
  c->K_global = K;
  CUDA_TRY(c.get(), cudaSetDevice(o.device));
  c->ks = N <= 3 ? get_kernels2d_a(N, M, o.dtype) : N <= 6 ? get_kernels2d_b(N, M, o.dtype) : get_kernels2d_c(N, M, o.dtype);
  if (!c->ks.launch_stage) return fail(nullptr, BBWADG_ERR_UNSUPPORTED, "no 2D kernel instantiation for this (N, M, dtype)");
  CUDA_TRY(c.get(), c->ks.prepare());
  int nsm = 0;
  CUDA_TRY(c.get(), cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, o.device));
  c->grid = nsm * c->ks.blocks_per_sm();
  c->stream = static_cast<cudaStream_t>(o.cuda_stream);
  Part& P = c->part;
  P.rank = 0;
  P.nparts = 1;
  P.K_local = K;
  P.n_interior = K;
  P.gid.resize(K);
  for (int64_t i = 0; i < K; ++i) P.gid[i] = i;
  P.nbr = nbr;
  P.code = code;
  P.send_off.assign(2, 0);
  P.recv_off.assign(2, 0);
  try {
    c->tables = build_tables_2d(N, M, (int)c->rb);
  } catch (const std::exception& ex) {
    return fail(nullptr, BBWADG_ERR_UNSUPPORTED, ex.what());
  }
  CUDA_TRY(c.get(), cudaMalloc(&c->d_tab, c->tables.blob.size()));
  CUDA_TRY(c.get(), cudaMemcpy(c->d_tab, c->tables.blob.data(), c->tables.blob.size(), cudaMemcpyHostToDevice));
  bbwadg_status st;
  if ((st = upload_real(c.get(), &c->d_geo, geo))) return fail(nullptr, st, c->err);
  if ((st = upload_real(c.get(), &c->d_c2, std::vector<double>(c2, c2 + (size_t)K * Mp)))) return fail(nullptr, st, c->err);
  CUDA_TRY(c.get(), cudaMalloc(&c->d_nbr, sizeof(int) * 3 * K));
  CUDA_TRY(c.get(), cudaMemcpy(c->d_nbr, nbr.data(), sizeof(int) * 3 * K, cudaMemcpyHostToDevice));
  CUDA_TRY(c.get(), cudaMalloc(&c->d_code, 3 * K));
  CUDA_TRY(c.get(), cudaMemcpy(c->d_code, code.data(), 3 * K, cudaMemcpyHostToDevice));
  const size_t sb = state_bytes(c.get());
  for (int b = 0; b < 2; ++b) {
    CUDA_TRY(c.get(), cudaMalloc(&c->d_Q[b], std::max<size_t>(sb, 16)));
    CUDA_TRY(c.get(), cudaMemset(c->d_Q[b], 0, sb));
  }
  CUDA_TRY(c.get(), cudaMalloc(&c->d_res, std::max<size_t>(sb, 16)));
  CUDA_TRY(c.get(), cudaMemset(c->d_res, 0, sb));
  CUDA_TRY(c.get(), cudaMalloc(&c->d_flag, sizeof(int)));
  CUDA_TRY(c.get(), cudaDeviceSynchronize());
  *out = c.release();
  return BBWADG_OK;
}

bbwadg_status bbwadg_setup_group(const bbwadg_mesh* mesh, int N, int M, const double* c2_coeffs,
                                 const bbwadg_options* opts, int nparts, bbwadg_ctx* out) {
  if (!out || nparts < 1) return fail(nullptr, BBWADG_ERR_INVALID_ARG, "bad group arguments");
  bbwadg_options o;
  bbwadg_default_options(&o);
  if (opts) o = *opts;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) return fail(nullptr, BBWADG_ERR_NO_DEVICE, "no CUDA device");
  GlobalMesh g;
  bbwadg_status s = prepare_global(mesh, N, M, c2_coeffs, &o, nparts, g);
  if (s) return s;
  Group* grp = new Group();
  cudaStream_t shared = nullptr;
  for (int r = 0; r < nparts; ++r) {
    bbwadg_ctx c = nullptr;
    s = setup_one(g, N, M, c2_coeffs, o, r, nparts, shared, &c);
    if (s) {
      // destroy the members built so far (the last one frees the group) and clear the caller's handles
      std::vector<bbwadg_ctx> built = grp->parts;
      for (auto p : built) bbwadg_destroy(p);
      if (built.empty()) delete grp;
      for (int j = 0; j < nparts; ++j) out[j] = nullptr;
      return s;
    }
    if (r == 0) {
      shared = c->stream;
      grp->stream = c->own_stream ? c->stream : nullptr;
      c->own_stream = false;
    }
    c->group = grp;
    c->group_index = r;
    grp->parts.push_back(c);
    out[r] = c;
  }
  return BBWADG_OK;
}

bbwadg_status bbwadg_set_state(bbwadg_ctx c, const void* Q, int on_device) {
  if (!c || !Q) return fail(c, BBWADG_ERR_INVALID_ARG, "null argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  size_t sb = state_bytes(c);
  CUDA_TRY(c, cudaMemcpyAsync(c->d_Q[c->cur], Q, sb, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                              c->stream));
  CUDA_TRY(c, cudaMemsetAsync(c->d_res, 0, sb, c->stream));
  if (!on_device) CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return BBWADG_OK;
}

bbwadg_status bbwadg_get_state(bbwadg_ctx c, void* Q, int on_device) {
  if (!c || !Q) return fail(c, BBWADG_ERR_INVALID_ARG, "null argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaMemcpyAsync(Q, c->d_Q[c->cur], state_bytes(c),
                              on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->stream));
  if (!on_device) CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return BBWADG_OK;
}

bbwadg_status bbwadg_set_source(bbwadg_ctx c, const double* gsrc) {
  if (!c) return fail(c, BBWADG_ERR_INVALID_ARG, "null ctx");
  if (c->elastic) return fail(c, BBWADG_ERR_UNSUPPORTED, "the manufactured source is acoustic only");
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (c->d_src) {
    CUDA_TRY(c, cudaFree(c->d_src));
    c->d_src = nullptr;
  }
  if (!gsrc) return BBWADG_OK;
  const Part& P = c->part;
  std::vector<double> loc((size_t)P.K_local * c->Np);
  for (int64_t i = 0; i < P.K_local; ++i)
    std::memcpy(&loc[(size_t)i * c->Np], gsrc + (size_t)P.gid[i] * c->Np, sizeof(double) * c->Np);
  return upload_real(c, &c->d_src, loc);
}

bbwadg_status bbwadg_rhs(bbwadg_ctx c, const void* Q_dev, double t, void* dQdt_dev) {
  if (!c || !Q_dev || !dQdt_dev) return fail(c, BBWADG_ERR_INVALID_ARG, "null argument");
  if (c->group) return fail(c, BBWADG_ERR_INVALID_ARG, "bbwadg_rhs is not available on group contexts");
  CUDA_TRY(c, cudaSetDevice(c->device));
  return full_pass(c, 1, Q_dev, dQdt_dev, 0, 0, 0, t);
}

bbwadg_status bbwadg_wadg_apply(bbwadg_ctx c, const void* r_dev, void* out_dev) {
  if (!c || !r_dev || !out_dev) return fail(c, BBWADG_ERR_INVALID_ARG, "null argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  return launch_pass(c, 2, r_dev, out_dev, 0, c->part.K_local, 0, 0, 0, 0);
}

bbwadg_status bbwadg_stage(bbwadg_ctx c, int s, double t, double dt) {
  if (!c || s < 0 || s > 4) return fail(c, BBWADG_ERR_INVALID_ARG, "bad arguments");
  if (c->group) return fail(c, BBWADG_ERR_INVALID_ARG, "use bbwadg_group_step for group contexts");
  CUDA_TRY(c, cudaSetDevice(c->device));
  bbwadg_status st = full_pass(c, 0, c->d_Q[c->cur], c->d_Q[1 - c->cur], RK_A[s], RK_B[s], dt, t + RK_C[s] * dt);
  if (st) return st;
  c->cur ^= 1;
  if (s == 4) {
    c->steps++;
    c->t = t + dt;
  }
  return BBWADG_OK;
}

bbwadg_status bbwadg_ipc_get_handles(bbwadg_ctx c, void* out) {
  if (!c || !out) return fail(c, BBWADG_ERR_INVALID_ARG, "null argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (!c->d_epoch) return fail(c, BBWADG_ERR_INVALID_ARG, "context is not a partitioned halo_transport 1 context");
  void* bufs[3] = {c->d_Q[0], c->d_Q[1], c->d_epoch};
  for (int b = 0; b < 3; ++b) {
    cudaIpcMemHandle_t h;
    CUDA_TRY(c, cudaIpcGetMemHandle(&h, bufs[b]));
    std::memcpy(static_cast<char*>(out) + 64 * b, &h, 64);
  }
  return BBWADG_OK;
}

bbwadg_status bbwadg_ipc_open_peer(bbwadg_ctx c, int peer, const void* handles) {
  if (!c || !handles || peer < 0 || peer >= c->part.nparts || peer >= 8)
    return fail(c, BBWADG_ERR_INVALID_ARG, "bad arguments");
  if (c->transport != 1) return fail(c, BBWADG_ERR_INVALID_ARG, "context was not set up with halo_transport 1");
  if (peer == c->part.rank) return fail(c, BBWADG_ERR_INVALID_ARG, "a rank does not open its own handles");
  if (c->peer_ipc[peer]) return BBWADG_OK;
  CUDA_TRY(c, cudaSetDevice(c->device));
  void* mapped[3] = {nullptr, nullptr, nullptr};
  for (int b = 0; b < 3; ++b) {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + 64 * b, 64);
    cudaError_t e = cudaIpcOpenMemHandle(&mapped[b], h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      for (int j = 0; j < b; ++j) cudaIpcCloseMemHandle(mapped[j]);
      return fail(c, BBWADG_ERR_CUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
    }
  }
  c->peer_q[peer][0] = mapped[0];
  c->peer_q[peer][1] = mapped[1];
  c->peer_epoch[peer] = static_cast<unsigned long long*>(mapped[2]);
  if (!c->d_sync_err) {
    CUDA_TRY(c, cudaMalloc(&c->d_sync_err, sizeof(int)));
    CUDA_TRY(c, cudaMemset(c->d_sync_err, 0, sizeof(int)));
  }
  c->peer_ipc[peer] = true;
  return BBWADG_OK;
}

bbwadg_status bbwadg_step(bbwadg_ctx c, double t, double dt) {
  if (!c) return fail(c, BBWADG_ERR_INVALID_ARG, "null ctx");
  if (c->group) return fail(c, BBWADG_ERR_INVALID_ARG, "use bbwadg_group_step for group contexts");
  CUDA_TRY(c, cudaSetDevice(c->device));
  for (int s = 0; s < 5; ++s) {
    bbwadg_status st = full_pass(c, 0, c->d_Q[c->cur], c->d_Q[1 - c->cur], RK_A[s], RK_B[s], dt, t + RK_C[s] * dt);
    if (st) return st;
    c->cur ^= 1;
  }
  c->steps++;
  c->t = t + dt;
  return BBWADG_OK;
}

bbwadg_status bbwadg_group_step(bbwadg_ctx* ctxs, int n, double t, double dt) {
  if (!ctxs || n < 1) return fail(nullptr, BBWADG_ERR_INVALID_ARG, "bad group");
  if (ctxs[0]->transport == 1) {
    // peer reads: every member reads the other members' Q_in in place; one shared stream orders stage s of
    // all members after stage s-1 of all members
    if (n > 8) return fail(ctxs[0], BBWADG_ERR_UNSUPPORTED, "peer-read halo: at most 8 partitions");
    for (int s = 0; s < 5; ++s) {
      for (int r = 0; r < n; ++r)
        for (int q = 0; q < n; ++q)
          for (int b = 0; b < 2; ++b) ctxs[r]->peer_q[q][b] = ctxs[q]->d_Q[b];
      for (int r = 0; r < n; ++r) {
        bbwadg_ctx c = ctxs[r];
        bbwadg_status st = launch_pass(c, 0, c->d_Q[c->cur], c->d_Q[1 - c->cur], 0, c->part.K_local, RK_A[s], RK_B[s],
                                       dt, t + RK_C[s] * dt);
        if (st) return st;
      }
      for (int r = 0; r < n; ++r) ctxs[r]->cur ^= 1;
    }
    for (int r = 0; r < n; ++r) {
      ctxs[r]->steps++;
      ctxs[r]->t = t + dt;
    }
    return BBWADG_OK;
  }
  for (int s = 0; s < 5; ++s) {
    // pack all partitions, then copy every ghost block from its owner's send buffer
    for (int r = 0; r < n; ++r) {
      bbwadg_ctx c = ctxs[r];
      int64_t ns = c->part.send_off.back();
      CUDA_TRY(c, c->ks.launch_pack(c->d_Q[c->cur], c->d_geo, c->d_sendfaces, (int)ns, fnode_ptr(c), c->d_send,
                                    c->stream));
    }
    for (int r = 0; r < n; ++r) {
      bbwadg_ctx c = ctxs[r];
      const size_t per_face = 2 * (size_t)c->Nfp * c->rb;
      for (int q = 0; q < n; ++q) {
        int64_t nr = c->part.recv_off[q + 1] - c->part.recv_off[q];
        if (nr == 0) continue;
        bbwadg_ctx peer = ctxs[q];
        int64_t ns = peer->part.send_off[r + 1] - peer->part.send_off[r];
        if (ns != nr) return fail(c, BBWADG_ERR_MESH, "halo size mismatch between partitions");
        CUDA_TRY(c, cudaMemcpyAsync(static_cast<char*>(c->d_ghost) + c->part.recv_off[q] * per_face,
                                    static_cast<char*>(peer->d_send) + peer->part.send_off[r] * per_face,
                                    nr * per_face, cudaMemcpyDeviceToDevice, c->stream));
      }
    }
    for (int r = 0; r < n; ++r) {
      bbwadg_ctx c = ctxs[r];
      const Part& P = c->part;
      bbwadg_status st = launch_pass(c, 0, c->d_Q[c->cur], c->d_Q[1 - c->cur], 0, P.n_interior, RK_A[s], RK_B[s], dt,
                                     t + RK_C[s] * dt);
      if (st) return st;
      st = launch_pass(c, 0, c->d_Q[c->cur], c->d_Q[1 - c->cur], P.n_interior, P.K_local, RK_A[s], RK_B[s], dt,
                       t + RK_C[s] * dt);
      if (st) return st;
    }
    for (int r = 0; r < n; ++r) ctxs[r]->cur ^= 1;
  }
  for (int r = 0; r < n; ++r) {
    ctxs[r]->steps++;
    ctxs[r]->t = t + dt;
  }
  return BBWADG_OK;
}

namespace {
// One LSRK step as a CUDA graph (the 5 stage launches captured on a private stream), for runs without a
// time-dependent source on single-partition contexts: replaying it removes the per-launch host overhead that
// dominates small meshes (DESIGN.md §6 "CUDA graph").  Two graphs, one per starting state buffer (a step
// flips the ping-pong buffers an odd number of times); rebuilt when dt changes.
bbwadg_status graph_run(bbwadg_ctx c, double t0, double dt, int64_t nsteps) {
  if (!c->gstream) {
    CUDA_TRY(c, cudaStreamCreateWithFlags(&c->gstream, cudaStreamNonBlocking));
    CUDA_TRY(c, cudaEventCreateWithFlags(&c->gev, cudaEventDisableTiming));
  }
  if (!c->gexec[0] || c->gdt != dt) {
    for (int b = 0; b < 2; ++b)
      if (c->gexec[b]) {
        cudaGraphExecDestroy(c->gexec[b]);
        c->gexec[b] = nullptr;
      }
    const int cur0 = c->cur;
    cudaStream_t user = c->stream;
    c->stream = c->gstream;  // launch_pass launches on c->stream
    for (int b = 0; b < 2; ++b) {
      c->cur = b;
      cudaGraph_t g = nullptr;
      cudaError_t e = cudaStreamBeginCapture(c->gstream, cudaStreamCaptureModeThreadLocal);
      bbwadg_status st = BBWADG_OK;
      for (int s = 0; e == cudaSuccess && st == BBWADG_OK && s < 5; ++s) {
        st = launch_pass(c, 0, c->d_Q[c->cur], c->d_Q[1 - c->cur], 0, c->part.K_local, RK_A[s], RK_B[s], dt,
                         RK_C[s] * dt);
        c->cur ^= 1;
      }
      cudaError_t e2 = cudaStreamEndCapture(c->gstream, &g);
      if (e == cudaSuccess) e = e2;
      if (e == cudaSuccess && st == BBWADG_OK) e = cudaGraphInstantiate(&c->gexec[b], g, 0);
      if (g) cudaGraphDestroy(g);
      if (st != BBWADG_OK || e != cudaSuccess) {
        c->stream = user;
        c->cur = cur0;
        if (st != BBWADG_OK) return st;
        return fail(c, BBWADG_ERR_CUDA, std::string("step graph: ") + cudaGetErrorString(e));
      }
    }
    c->stream = user;
    c->cur = cur0;
    c->gdt = dt;
  }
  CUDA_TRY(c, cudaEventRecord(c->gev, c->stream));
  CUDA_TRY(c, cudaStreamWaitEvent(c->gstream, c->gev, 0));
  for (int64_t i = 0; i < nsteps; ++i) {
    CUDA_TRY(c, cudaGraphLaunch(c->gexec[c->cur], c->gstream));
    c->cur ^= 1;  // 5 stages = an odd number of buffer flips
  }
  CUDA_TRY(c, cudaEventRecord(c->gev, c->gstream));
  CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->gev, 0));
  c->steps += nsteps;
  c->t = t0 + nsteps * dt;
  return BBWADG_OK;
}
}  // namespace

bbwadg_status bbwadg_run(bbwadg_ctx c, double t0, double dt, int64_t nsteps) {
  if (!c || nsteps < 0) return fail(c, BBWADG_ERR_INVALID_ARG, "bad arguments");
  if (c->group) return fail(c, BBWADG_ERR_INVALID_ARG, "use bbwadg_group_step for group contexts");
  const bool graphable = nsteps >= 2 && c->part.nparts == 1 && !c->d_src && !getenv("BBWADG_NO_GRAPH");
  if (graphable) {
    CUDA_TRY(c, cudaSetDevice(c->device));
    bbwadg_status s = graph_run(c, t0, dt, nsteps);
    if (s) return s;
  } else {
    for (int64_t i = 0; i < nsteps; ++i) {
      bbwadg_status s = bbwadg_step(c, t0 + i * dt, dt);
      if (s) return s;
    }
  }
  CUDA_TRY(c, cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
  long long n = (long long)c->part.K_local * c->nfields * c->Np;
  if (n > 0) {
    if (c->dtype == BBWADG_F64)
      nonfinite_kernel<double><<<592, 256, 0, c->stream>>>(static_cast<const double*>(c->d_Q[c->cur]), n, c->d_flag);
    else
      nonfinite_kernel<float><<<592, 256, 0, c->stream>>>(static_cast<const float*>(c->d_Q[c->cur]), n, c->d_flag);
    CUDA_TRY(c, cudaGetLastError());
  }
  int flag = 0, serr = 0;
  CUDA_TRY(c, cudaMemcpyAsync(&flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  if (c->d_sync_err) CUDA_TRY(c, cudaMemcpyAsync(&serr, c->d_sync_err, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (serr) return fail(c, BBWADG_ERR_CUDA, "peer stage barrier timed out (a peer stopped advancing)");
  if (c->comm) {
    const int ne = nccl::async_error(c->comm);
    if (ne != 0 && ne != 7) {
      std::ostringstream os;
      os << "NCCL asynchronous error " << ne << " (" << nccl::last_error(c->comm) << ")";
      return fail(c, BBWADG_ERR_NCCL, os.str());
    }
  }
  if (flag) {
    std::ostringstream os;
    os << "non-finite state after step " << c->steps;
    return fail(c, BBWADG_ERR_NONFINITE, os.str());
  }
  return BBWADG_OK;
}

bbwadg_status bbwadg_synchronize(bbwadg_ctx c) {
  if (!c) return fail(c, BBWADG_ERR_INVALID_ARG, "null ctx");
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (c->comm) {
    const int ne = nccl::async_error(c->comm);
    if (ne != 0 && ne != 7) return fail(c, BBWADG_ERR_NCCL, std::string("NCCL asynchronous error: ") + nccl::last_error(c->comm));
  }
  return BBWADG_OK;
}

bbwadg_status bbwadg_query(bbwadg_ctx c, bbwadg_info* info) {
  if (!c || !info) return fail(c, BBWADG_ERR_INVALID_ARG, "null argument");
  const Part& P = c->part;
  info->num_elements_global = c->K_global;
  info->num_elements_local = P.K_local;
  info->num_interior_local = P.n_interior;
  info->num_halo_faces = P.num_ghost();
  info->N = c->N;
  info->M = c->M;
  info->Np = c->Np;
  info->Mp = c->Mp;
  info->dtype = c->dtype;
  info->rank = P.rank;
  info->world_size = P.nparts;
  info->global_ids = P.gid.data();
  // minimum HBM traffic of one fused stage: Q_in, res (read) + Q_out, res (write) = 16 Np words,
  // c^2_M (Mp words), geometry (12 words), connectivity (4 int32 + 4 bytes) per element.
  const double per_elem = c->elastic ? (36.0 * c->Np + 3.0 * c->Mp + 12.0) * c->rb + 20.0
                         : c->dim == 2 ? (12.0 * c->Np + c->Mp + 6.0) * c->rb + 15.0
                                       : (16.0 * c->Np + c->Mp + 12.0) * c->rb + 20.0;
  info->algorithmic_bytes_per_stage = per_elem * P.K_local;
  const int N = c->N, M = c->M, Np = c->Np, Nfp = c->Nfp;
  double vol = 24.0 * np3(N - 1) + 8.0 * Np * 4;                  // gradient (24 flop/b) + elevation (8 flop/out)
  double surf = 4.0 * (Nfp * 20.0 + 2 * Nfp * 14.0 + 2 * 6.0 * np3(N - 1) + 16.0 * Np / 4.0 * 4.0);
  double mult = 2.0 * Np * c->Mp + np3(N + M);
  double proj = 0;
  for (int n = N + 1; n <= N + M; ++n) proj += 8.0 * np3(n - 1);
  for (int n = 1; n <= N; ++n) proj += 8.0 * np3(n - 1) + 10.0 * np3(n);
  double lsrk = 4.0 * 4 * Np;
  if (c->dim == 2) {
    // 2D: gradient 3 x 3 x 2 flop per degree-(N-1) coefficient + elevation; fluxes, 6 edge lifts (N layers of
    // 2-point sums); product 2 Np Mp; projection 6 flop per reduction output, 8 per upward output; LSRK
    const int Nfp2 = N + 1;
    vol = 18.0 * (N * (N + 1) / 2) + 3.0 * 3 * Np;
    surf = 3.0 * (Nfp2 * 20.0) + 6.0 * (3.0 * Nfp2 + 3.0 * Np);
    mult = 2.0 * Np * c->Mp;
    proj = 0;
    for (int n = N + 1; n <= N + M; ++n) proj += 3.0 * (n * (n + 1) / 2);
    for (int n = 1; n <= N; ++n) proj += 3.0 * (n * (n + 1) / 2) + 5.0 * ((n + 1) * (n + 2) / 2);
    lsrk = 4.0 * 3 * Np;
  }
  if (c->elastic) {
    // 9-field gradient (144 flop per degree-(N-1) coefficient) + 9 elevations; fluxes (~90 flop per face
    // node) + three 8-array lifts; ten scalar WADG applications; LSRK on 9 fields
    vol = 144.0 * np3(N - 1) + 9.0 * 4 * Np;
    surf = 4.0 * Nfp * 90.0 + 3.0 * (surf - 4.0 * Nfp * 20.0);
    mult *= 10.0;
    proj *= 10.0;
    lsrk = 4.0 * 9 * Np;
  }
  info->flops_per_stage = (vol + surf + mult + proj + lsrk) * P.K_local;
  info->kernels_per_stage = (P.nparts > 1) ? 3 : 1;
  info->steps_taken = c->steps;
  info->time = c->t;
  return BBWADG_OK;
}

const char* bbwadg_error_string(bbwadg_ctx c) { return c ? c->err.c_str() : g_last_error.c_str(); }
const char* bbwadg_last_error(void) { return g_last_error.c_str(); }

void bbwadg_destroy(bbwadg_ctx c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (int r = 0; r < 8; ++r)
    if (c->peer_ipc[r]) {
      for (int b = 0; b < 2; ++b)
        if (c->peer_q[r][b]) cudaIpcCloseMemHandle(c->peer_q[r][b]);
      if (c->peer_epoch[r]) cudaIpcCloseMemHandle(c->peer_epoch[r]);
    }
  void* bufs[] = {c->d_tab, c->d_Q[0], c->d_Q[1], c->d_res, c->d_c2, c->d_geo, c->d_nbr, c->d_code,
                  c->d_src, c->d_ghost, c->d_send, c->d_sendfaces, c->d_flag, c->d_qctr, c->d_ptime, c->d_gmap,
                  c->d_epoch, c->d_sync_err};
  for (void* p : bufs)
    if (p) cudaFree(p);
  for (int b = 0; b < 2; ++b)
    if (c->gexec[b]) cudaGraphExecDestroy(c->gexec[b]);
  if (c->gev) cudaEventDestroy(c->gev);
  if (c->gstream) cudaStreamDestroy(c->gstream);
  if (c->comm) nccl::comm_destroy(c->comm);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->ev_ready) cudaEventDestroy(c->ev_ready);
  if (c->ev_halo) cudaEventDestroy(c->ev_halo);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  if (c->group) {
    Group* g = c->group;
    auto it = std::find(g->parts.begin(), g->parts.end(), c);
    if (it != g->parts.end()) g->parts.erase(it);
    if (g->parts.empty()) {
      if (g->stream) cudaStreamDestroy(g->stream);
      delete g;
    }
  }
  delete c;
}

bbwadg_status bbwadg_partition_plan(const bbwadg_mesh* mesh, int nparts, const int cuts[3], int rank, int64_t* sizes,
                                    int64_t* gid, int64_t* send, int64_t* recv) {
  if (!mesh || !mesh->vertices || !mesh->elements || nparts < 1 || rank < 0 || rank >= nparts || !sizes)
    return fail(nullptr, BBWADG_ERR_INVALID_ARG, "bad arguments");
  GlobalMesh g;
  g.K = mesh->num_elements;
  g.nv = mesh->num_vertices;
  g.V = mesh->vertices;
  g.EV = mesh->elements;
  std::string e = check_orientation(g);
  if (e.empty()) e = build_connectivity(g);
  if (!e.empty()) return fail(nullptr, BBWADG_ERR_MESH, e);
  e = partition(g, nparts, cuts);
  if (!e.empty()) return fail(nullptr, BBWADG_ERR_INVALID_ARG, e);
  Part P = build_part(g, rank, nparts);
  const int64_t ns = P.send_off.back(), ng = P.num_ghost();
  sizes[0] = P.K_local;
  sizes[1] = P.n_interior;
  sizes[2] = ns;
  sizes[3] = ng;
  if (gid) std::copy(P.gid.begin(), P.gid.end(), gid);
  if (send) {
    for (int r = 0; r < nparts; ++r)
      for (int64_t i = P.send_off[r]; i < P.send_off[r + 1]; ++i) {
        int64_t k = P.gid[P.send_faces[2 * i]];
        int f = P.send_faces[2 * i + 1];
        send[4 * i] = k;
        send[4 * i + 1] = f;
        send[4 * i + 2] = r;
        send[4 * i + 3] = g.etoe[4 * k + f];
      }
  }
  if (recv) {
    for (int64_t i = 0; i < P.K_local; ++i)
      for (int f = 0; f < 4; ++f) {
        int nb = P.nbr[4 * i + f];
        if (nb > -2) continue;
        int64_t slot = -2 - (int64_t)nb;
        int src = 0;
        while (P.recv_off[src + 1] <= slot) ++src;
        int64_t k = P.gid[i];
        recv[4 * slot] = k;
        recv[4 * slot + 1] = f;
        recv[4 * slot + 2] = src;
        recv[4 * slot + 3] = g.etoe[4 * k + f];
      }
  }
  return BBWADG_OK;
}

bbwadg_status bbwadg_projection_constants(int N, int M, double* out) {
  if (!out || N < 0 || N > 30 || M < 0) return fail(nullptr, BBWADG_ERR_INVALID_ARG, "bad arguments");
  auto c = projection_constants(N, M);
  std::copy(c.begin(), c.end(), out);
  return BBWADG_OK;
}

bbwadg_status bbwadg_mass_inverse_constants(int N, double* out) {
  if (!out || N < 0 || N > 30) return fail(nullptr, BBWADG_ERR_INVALID_ARG, "bad arguments");
  auto c = mass_inverse_constants(N);
  std::copy(c.begin(), c.end(), out);
  return BBWADG_OK;
}

bbwadg_status bbwadg_nccl_unique_id(void* out) {
  if (!out) return fail(nullptr, BBWADG_ERR_INVALID_ARG, "null out");
  std::string why;
  if (!nccl::load(why)) return fail(nullptr, BBWADG_ERR_NCCL, why);
  if (nccl::get_unique_id(out) != 0) return fail(nullptr, BBWADG_ERR_NCCL, "ncclGetUniqueId failed");
  return BBWADG_OK;
}

// Debug/test hook (not in the public header): copy the host table blob of (N, M, fp_bytes).
// offsets[0..11] = byte offsets (up, dn, dec, fnode, nbrvol, nbrface, triup, l0, lgather, invfactN,
// invfactM, post); returns the blob size, copies min(size, cap) bytes into out when out != NULL.
int64_t bbwadg_debug_tables(int N, int M, int fp_bytes, void* out, int64_t cap, double* gam, double* lam) {
  HostTables T;
  try {
    T = build_tables(N, M, fp_bytes);
  } catch (...) {
    return -1;
  }
  if (gam)
    for (int j = 0; j <= N; ++j) gam[j] = T.gam[j];
  if (lam)
    for (int j = 0; j <= N; ++j) lam[j] = T.lam[j];
  if (out) std::memcpy(out, T.blob.data(), std::min<size_t>(T.blob.size(), (size_t)cap));
  return (int64_t)T.blob.size();
}

// Debug hook (not in the public header): per-phase cycle counters accumulated by a
// BBW_PHASE_TIMING build when BBWADG_PHASE_TIMING is set; copies 32 values, resets them.
int bbwadg_debug_phase_times(bbwadg_ctx c, unsigned long long* out) {
  if (!c || !c->d_ptime || !out) return -1;
  cudaStreamSynchronize(c->stream);
  cudaMemcpy(out, c->d_ptime, 32 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  cudaMemset(c->d_ptime, 0, 32 * sizeof(unsigned long long));
  return 0;
}

const char* bbwadg_version(void) { return "bbwadg-b200 0.2 (sm_100a, fused acoustic stage kernel v5, elastic stage kernel e1)"; }

}  // extern "C"
