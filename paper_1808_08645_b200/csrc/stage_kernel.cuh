// Fused BBWADG RK-stage kernel for sm_100a, v3 (templated on N, M, the real type and the
// group shape).
//
// Work decomposition.  A CTA of T threads is split into G independent GROUPS of TG threads
// (TG a multiple of 32).  Each group processes batches of ET consecutive elements (Morton order:
// neighbour traces are mostly L2-resident) and synchronises only with itself (named barrier
// `bar.sync 1+g, TG`, or __syncwarp when TG == 32), so the latency chains of different groups
// overlap.  Within a group, thread q "owns" canonical coefficients a = q + TG k: its copies of
// Q_in, of the LSRK residual and of r_u live in REGISTERS (the residual is loaded at batch start
// and only consumed at the end, hiding its HBM latency); shared memory only holds the arrays
// that stencils gather from, with the surface and WADG work regions aliased.
//
// Per-output index work is amortised: a thread computes output i of a phase for its group's ET
// elements (and, on faces, for all 8 face/flux arrays) from one table lookup; every shared
// address is "table register + compile-time immediate".  One-degree Bernstein reductions and
// elevations are UNWEIGHTED sums in factorial-scaled variables (layout.hpp).
//   A  Q_in -> smem (16-B vectors); residual -> registers; c^2_M/b!; grad(lambda), normals
//   B  own Q -> registers; fluxes F_p, F_u x |grad l_f| c!;
//      g''_b = sum_i grad(l_i) q_{b+e_i} / b!                       (barycentric derivative)
//   C  r''_a = -sum_j g''_{a-e_j} (volume); L_0 F: reduction, 1/(d!)^2, elevation, (c!)^2
//   D  N face reductions -> lift layers
//   E  gather the 4 lifts; LSRK update of u (registers -> HBM)
//   F  Bernstein product h'_g = (g!)^2 N!M!/(N+M)! sum r''_a c''_b        (Eq. mcoeff)
//   G  M reductions N+M -> N; H N downward reductions; I N upward elevations with level
//      constants gam_n = (n!)^2 c_{N-n}/(N+M)!                        (Eq. telescope)
//   J  dp/dt_a = a!/N! b_N[a]; LSRK update of p
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "layout.hpp"

namespace bbw {

__host__ __device__ constexpr int cnp3(int n) { return lnp3(n); }
__host__ __device__ constexpr int cnp2(int n) { return lnp2(n); }
__host__ __device__ constexpr int cnp4(int n) { return lnp4(n); }
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }
__host__ __device__ constexpr int rup(int a, int b) { return (a + b - 1) / b * b; }

template <typename R>
struct StageArgs {
  const R* Qin;
  R* Qout;
  R* res;
  const R* c2;
  const R* geo;        // [K][12]: grad(lambda_0..3)
  const int* nbr;      // [K][4]
  const uint8_t* code; // [K][4] = 6 f' + sigma
  const R* ghost;      // [slots][2][NFP]: p and u.n_sender at the sender's face nodes (halo, Eq. sdf)
  // peer-read halo (halo_transport 1): the stage inputs Q_in of the other partitions (same device, or mapped
  // from other processes / GPUs by CUDA IPC over NVLink), indexed by owner rank; gmap[slot] = (owner rank,
  // owner-local element id) of ghost slot `slot`.  Partition faces then read the neighbour's traces directly
  // (no pack, no collective) with the interior-face arithmetic, so partitioned runs are bitwise equal to
  // the single-partition run.
  const R* peer[8];
  const int* gmap;
  const R* src;        // [K][NP] or null
  const uint8_t* tab;  // table blob (layout.hpp)
  unsigned int* qctr;  // BBW_DYNQ work queue [2] (zero at launch; the kernel's last unit resets it)
  int qch;             // unit-batches per work-queue ticket (>= 1; the host picks it from the batches per unit)
  long long elem_begin, elem_end;
  R rk_a, rk_b, dt, src_amp, tau_p, tau_u;
  R gam[10], lam[10];
  int mode;  // 0 LSRK stage, 1 write dQ/dt into Qout, 2 WADG apply (Qin=r[K][NP] -> Qout[K][NP])
  unsigned long long* ptime;  // BBW_PHASE_TIMING builds only: per-phase cycle counters [32]
};

#ifndef BBW_T
#define BBW_T 128
#endif
#ifndef BBW_DEFER_ST
#define BBW_DEFER_ST 1  // sparse phases: all outputs' loads before the stores (no store between loads)
#endif

// default group shape per N: threads per group and elements per group-batch
// default group shape per N (A/B-measured, scripts/ab_subwarp*.sh): sub-warp groups of TG = 4 / 4 / 8 / 16
// lanes per element for N = 1..4 (2.2x, 1.5x, 1.07x, 1.02x over whole-warp groups with 4 / 4 / 2 / 2
// elements per lane), one warp per element for N = 5..7, two for N = 8, 9
__host__ __device__ constexpr int default_tg(int N) { return N <= 2 ? 4 : N == 3 ? 8 : N == 4 ? 16 : N <= 7 ? 32 : 64; }
__host__ __device__ constexpr int default_et(int N) { return N > 0 ? 1 : 1; }
// minimum resident CTAs per SM for __launch_bounds__ (caps registers at 65536 / (T * MINB)); A/B-measured
// (scripts/ab_minb.sh): 5 for N = 4, 5 (+3.6 %, +2..3 %), 4 elsewhere (N=6: -5.7 %, N=7: -15 % at 5)
__host__ __device__ constexpr int default_minb(int N) { return (N == 4 || N == 5) ? 5 : 4; }

#ifndef BBW_ROWD
#define BBW_ROWD 0  // row-owned lift layers (phase D): measured -13 % at (7,4), -19 % at (5,3), -42 % at (9,9) (spills)
#endif
#ifndef BBW_FPAD
#define BBW_FPAD 2  // face-array padding (reals) for the row-owned layer sweep
#endif

#ifndef BBW_TRIPLE
#define BBW_TRIPLE 2  // shell-order ownership of the WADG projection: 1 always, 0 never, 2 where it measured faster
#endif

template <int N_, int M_, typename R>
struct StageCfg {
  static constexpr int N = N_, M = M_;
  static constexpr int NP = cnp3(N), NFP = cnp2(N), NFP1 = cnp2(N - 1), MP = cnp3(M), NPH = cnp3(N + M);
  static constexpr int NPM1 = cnp3(N - 1), NP4 = cnp4(N);
  static constexpr int RB = (int)sizeof(R);
  static constexpr int VEC = 16 / RB;
  static constexpr int T = BBW_T;
#ifdef BBW_TG
  static constexpr int TG = BBW_TG;
#else
  static constexpr int TG = default_tg(N);
#endif
#ifdef BBW_ET
  static constexpr int ET = BBW_ET;
#else
  static constexpr int ET = default_et(N);
#endif
#ifdef BBW_MINB
  static constexpr int MINB = BBW_MINB;
#else
  // fp32 (half the element block): 6 CTAs per SM for the whole-warp groups of N = 5..7 (A/B: +9.3 % at (7,4),
  // +1.9 % at (5,3); 8 CTAs spills and is slower), the fp64 choice elsewhere
  static constexpr int MINB = (sizeof(R) == 4 && N >= 5 && N <= 7) ? 6 : default_minb(N);
#endif
  static constexpr bool DEFER = BBW_DEFER_ST != 0;  // sparse phases store after all loads (elastic: off, measured)
  static constexpr int G = T / TG;               // groups per CTA
  static constexpr int KO = (NP + TG - 1) / TG;  // owned coefficients per thread
  // ---- per-element shared-memory layout (in reals)
  static constexpr int O_GEO = 0, O_C = 40, O_RP = 40 + MP;  // GEO: grad l (12), normals+|grad l| (16), nbr/code ints
  static constexpr int O_X = rup(O_RP + NP, VEC);
  static constexpr int X_Q = O_X, X_G = O_X + 4 * NP, X_L = O_X;  // Q + G'', later the lift layers
  // lift-layer arrays: 8 face/flux arrays of NP reals (layers j = 0..N concatenated) at stride FS; the
  // row-owned layer sweep (BBW_ROWD) pads FS so the 8 arrays start in different shared-memory banks
  static constexpr bool ROWD = BBW_ROWD && TG >= 32 && ET == 1;
  static constexpr int FS = ROWD ? NP + BBW_FPAD : NP;
  static constexpr int XSIZE = cmax(4 * NP + 4 * (NPM1 + 1), 8 * FS);
  static constexpr int O_Y = O_X + XSIZE;
  static constexpr int Y_F = O_Y, Y_Y = O_Y + 8 * NFP;  // F', Y''
  // zero-padded rows of r''_p for the product: row (a2,a3) at rowid * RS (RS = N+1 rounded up to an
  // odd number of 16-B vectors, against bank conflicts), then one all-zero row; written in E, read by F
  static constexpr int RS = rup(N + 1, VEC) + ((rup(N + 1, VEC) / VEC) % 2 == 0 ? VEC : 0);  // odd # of vectors
  static constexpr int NS = (NFP + 1) * RS;
  static constexpr int YSIZE = cmax(cmax(8 * NFP + 8 * (NFP1 + 1), NS), 0);
  static constexpr int Y_RPP = O_Y;
  // WADG work arrays (alias X, Y): h (degree N+M) at W_H, the reduction ping-pong partner (degree
  // N+M-1) at W_P, and the N+1 levels of the telescoping sweeps, level n at lev(n) with one zero slot
  // just before it; the upward sweep overwrites u_n by b_n in place.  The levels are placed in the
  // region the LAST M-reduction does not read, so they alias h / P as well.
  static constexpr int NPH1 = cnp3(N + M - 1);
  static constexpr int LEVSZ = NP4 + N + 1;
  static constexpr bool LAST_FROM_H = (M >= 1) && ((M - 1) % 2 == 0);
  // ALIAS only when the WADG arrays would set the element's smem size (high N, M); otherwise the
  // round-1 v3 layout (separate levels, ping-pong upward buffers A0/A1) is kept: measured ~2 % faster.
  static constexpr int W_H = O_X, W_P = W_H + NPH;
  static constexpr int WSIZE_V3 = 2 * NPH + NP4 + 2 * (NP + 1);
  static constexpr bool ALIAS = WSIZE_V3 > XSIZE + YSIZE;
  static constexpr int W_LEV = !ALIAS ? W_P + NPH : (M == 0 || LAST_FROM_H) ? W_P : (LEVSZ <= NPH ? W_H : W_P + NPH1);
  static constexpr int W_A0 = W_LEV + NP4, W_A1 = W_A0 + NP + 1;  // !ALIAS only
  static constexpr int WSIZE = !ALIAS ? WSIZE_V3
                                      : cmax(cmax(W_LEV + LEVSZ, W_P + (M >= 1 ? NPH1 : 0)), W_H + NPH) - O_X;
  static __host__ __device__ constexpr int lev(int n) { return ALIAS ? W_LEV + lnp4(n - 1) + n + 1 : W_LEV + lnp4(n - 1); }
  // shell-order ("triple") WADG layout (BBW_TRIPLE): product output h (degree N+M) at T_H, the G ping-pong
  // partner at T_P, the N+1 levels of the telescoping sweeps at tlev(n) (each preceded by a zero slot),
  // placed over a region that is dead when G's last step writes level N
  static constexpr int T_H = O_X, T_P = T_H + NPH, T_LEVSZ = NP4 + N + 1;
  static constexpr bool T_LAST_FROM_P = (M >= 1) && ((M - 1) % 2 == 1);
  static constexpr int T_LVB = (M == 0) ? O_X
                               : (M == 1) ? T_P
                               : T_LAST_FROM_P ? (T_LEVSZ <= NPH ? T_H : T_P + NPH1)
                                               : (T_LEVSZ <= NPH1 ? T_P : T_P + NPH1);
  static __host__ __device__ constexpr int tlev(int n) { return T_LVB + lnp4(n - 1) + n + 1; }
  static constexpr int T_WSIZE = cmax(cmax(T_LVB + T_LEVSZ, T_P + (M >= 1 ? NPH1 : 0)), T_H + NPH) - O_X;
  // A/B (scripts/gpu_r2_full.sh): +18 % at N = M = 9, +2 % at (5,3), -3 % at (7,4) and (3,1) -> used for N+M >= 14
  static constexpr bool TRIPLE = BBW_TRIPLE == 1 ? true : BBW_TRIPLE == 0 ? false : (N + M >= 14);
  static constexpr int PER_E = rup(O_X + cmax(XSIZE + YSIZE, TRIPLE ? T_WSIZE : WSIZE), VEC);
  static constexpr int EB = PER_E * RB;  // element stride in bytes
  static constexpr int GB = ET * EB;     // group stride in bytes
  static constexpr int SMEM_BYTES = G * GB + 16 * G;  // + one mbarrier and one work-queue ticket per group
  static constexpr int GPW = TG < 32 ? 32 / TG : 1;  // groups per warp (sub-warp groups for small N)
  static_assert((TG % 32 == 0 || 32 % TG == 0) && T % TG == 0 && (TG <= 32 || G <= 15), "bad group shape");
};

template <class C>
struct GroupSync {
  int id;
  __device__ __forceinline__ void operator()() const {
    if constexpr (C::TG <= 32) {  // sub-warp groups of one warp run the same phase sequence in lockstep
      __syncwarp();
    } else {
      asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(C::TG) : "memory");
    }
  }
};

#ifdef BBW_PHASE_TIMING
#define BBW_PT(id)                                                     \
  do {                                                                 \
    if (q == 0 && A.ptime) {                                           \
      const long long t_ = clock64();                                  \
      atomicAdd(A.ptime + (id), (unsigned long long)(t_ - pt_prev));   \
      pt_prev = t_;                                                    \
    }                                                                  \
  } while (0)
#else
#define BBW_PT(id) \
  do {             \
  } while (0)
#endif

// switch (n) { case 10: f(9); case 9: f(8); ... case 1: f(0); } with fall-through: runs f(n-1..0)
#define BBW_FALLTHROUGH_SWITCH(n, f)                   \
  switch (n) {                                         \
    case 10: f(std::integral_constant<int, 9>{}); [[fallthrough]]; \
    case 9: f(std::integral_constant<int, 8>{}); [[fallthrough]];  \
    case 8: f(std::integral_constant<int, 7>{}); [[fallthrough]];  \
    case 7: f(std::integral_constant<int, 6>{}); [[fallthrough]];  \
    case 6: f(std::integral_constant<int, 5>{}); [[fallthrough]];  \
    case 5: f(std::integral_constant<int, 4>{}); [[fallthrough]];  \
    case 4: f(std::integral_constant<int, 3>{}); [[fallthrough]];  \
    case 3: f(std::integral_constant<int, 2>{}); [[fallthrough]];  \
    case 2: f(std::integral_constant<int, 1>{}); [[fallthrough]];  \
    case 1: f(std::integral_constant<int, 0>{}); [[fallthrough]];  \
    default: break;                                    \
  }


__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem)
               : "memory");
}
template <typename R>
__device__ __forceinline__ void cp_async_real(void* smem, const R* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem),
               "n"((int)sizeof(R))
               : "memory");
}
// TMA bulk copies (cp.async.bulk, SASS UBLKCP) completing on a per-group mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* mbar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(mbar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* mbar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(mbar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes, uint64_t* mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(mbar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mbar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @P1 bra DONE;\n bra LAB_WAIT;\n DONE:\n}" ::"r"((unsigned)__cvta_generic_to_shared(mbar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

#ifndef BBW_PF  // L2 prefetch of the next batch: no speed-up measured, +7 GB DRAM reads per config-5 stage
#define BBW_PF 0
#endif
#ifndef BBW_M0_FAST
#define BBW_M0_FAST 1  // M = 0: WADG = multiplication by the constant c^2 (skip the product and the sweeps)
#endif
#ifndef BBW_LSRK_TMEM
#define BBW_LSRK_TMEM 0
#endif
#ifndef BBW_LSRK_REG
#define BBW_LSRK_REG 1
#endif
#ifndef BBW_CPASYNC
#define BBW_CPASYNC 1
#endif
#ifndef BBW_TMA
#define BBW_TMA 1  // element Q blocks, geometry and neighbour ids by cp.async.bulk (needs BBW_CPASYNC)
#endif
#ifndef BBW_FLUX_LATE
#define BBW_FLUX_LATE 0  // fluxes (B1b) after C1: measured -6 % at (7,4) and -5 % at (5,3) (register spills; rejected)
#endif
#ifndef BBW_DYNQ
#define BBW_DYNQ 1  // batches handed out by a global atomic ticket (tight in-flight window: neighbour traces hit L2)
#endif
#ifndef BBW_TMA_MIN_TG
#define BBW_TMA_MIN_TG 32  // TMA only for whole-warp groups (sub-warp groups: cp.async; see the kernel)
#endif

// predicated 16-B shared load into x[0..VEC): registers keep their old values when !p
template <typename R, int OFF>
__device__ __forceinline__ void ld_shared_vec_pred(R* x, unsigned addr, bool p) {
  if constexpr (sizeof(R) == 8) {
    asm("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.shared.v2.f64 {%0, %1}, [%3+%4];\n}\n"
        : "+d"(x[0]), "+d"(x[1])
        : "r"((int)p), "r"(addr), "n"(OFF));
  } else {
    asm("{\n .reg .pred q;\n setp.ne.b32 q, %4, 0;\n @q ld.shared.v4.f32 {%0, %1, %2, %3}, [%5+%6];\n}\n"
        : "+f"(x[0]), "+f"(x[1]), "+f"(x[2]), "+f"(x[3])
        : "r"((int)p), "r"(addr), "n"(OFF));
  }
}

// (x!)^2 as a compile-time constant (exact integer factorial, one rounding)
__host__ __device__ constexpr double fact2c(int x) {
  double f = 1.0;
  for (int i = 2; i <= x; ++i) f *= i;
  return f * f;
}

// unpredicated 16-B shared load into x[0..VEC) (opaque to the compiler, so x stays in registers)
template <typename R, int OFF>
__device__ __forceinline__ void ld_shared_vec(R* x, unsigned addr) {
  if constexpr (sizeof(R) == 8) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+%3];\n" : "+d"(x[0]), "+d"(x[1]) : "r"(addr), "n"(OFF));
  } else {
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4+%5];\n"
                 : "+f"(x[0]), "+f"(x[1]), "+f"(x[2]), "+f"(x[3])
                 : "r"(addr), "n"(OFF));
  }
}

// smallest g2 + g3 among the product output rows of a pass starting at ROWDEC entry r0: ROWDEC is sorted
// by s = g2 + g3 and only permuted inside 32-row blocks (tables.cpp), so it is the s of row 32*floor(r0/32)
__host__ __device__ constexpr int prod_pass_smin(int r0) {
  int b = r0 / 32 * 32, s = 0;
  while ((s + 1) * (s + 2) / 2 <= b) ++s;
  return s;
}
__host__ __device__ constexpr int prod_acc_off(int nm, int tg, int k) {
  int o = 0;
  for (int j = 0; j < k; ++j) o += nm + 1 - prod_pass_smin(tg * j);
  return o;
}
__host__ __device__ constexpr int prod_acc_total(int nm, int tg, int kr) { return prod_acc_off(nm, tg, kr); }
#ifndef BBW_PROD_V5
#define BBW_PROD_V5 1
#endif
#ifndef BBW_PROD_SWITCH
#define BBW_PROD_SWITCH 0  // measured 4-6 % slower than the predicated loads + branches
#endif

// LSRK outputs (Q_out, residual): streaming stores (evict-first), so the L2 keeps the stage input
// Q_in that neighbour face traces are read from
#ifndef BBW_STCS
#define BBW_STCS 0  // measured: no DRAM saving, -0.6 % at N=7
#endif
template <typename R>
__device__ __forceinline__ void st_out(R* p, R v) {
#if BBW_STCS
  __stcs(p, v);
#else
  *p = v;
#endif
}

template <typename R>
__device__ __forceinline__ R ld(const char* p) { return *reinterpret_cast<const R*>(p); }
template <typename R>
__device__ __forceinline__ void st(char* p, R v) { *reinterpret_cast<R*>(p) = v; }

template <int I, int END, int STEP, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr ((STEP > 0 && I < END) || (STEP < 0 && I > END)) {
    f(std::integral_constant<int, I>{});
    static_for<I + STEP, END, STEP>(f);
  }
}

// ---- TMEM (tensor memory) as lane-private storage for the LSRK state (BBW_LSRK_TMEM): each lane keeps
// its Q_in copy and residual in its own TMEM lane between the batch start and phases E / J, so those 64
// registers are free for the sparse phases (SASS STTM / LDTM; TMEM traffic does not use L1 wavefronts)
template <int NW>
__device__ __forceinline__ void tm_st(uint32_t taddr, const uint32_t* v);
template <>
__device__ __forceinline__ void tm_st<8>(uint32_t t, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(t), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
template <>
__device__ __forceinline__ void tm_st<16>(uint32_t t, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(t),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
template <int NW>
__device__ __forceinline__ void tm_ld(uint32_t taddr, uint32_t* v);
template <>
__device__ __forceinline__ void tm_ld<8>(uint32_t t, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(t)
               : "memory");
}
template <>
__device__ __forceinline__ void tm_ld<16>(uint32_t t, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(t)
      : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// store / load n reals (n*RB/4 32-bit columns, in chunks of 16 / 8 columns) at column offset col
template <typename R, int NR>
__device__ __forceinline__ void tm_store_reals(uint32_t taddr, int col0, const R* x) {
  constexpr int NWD = NR * (int)sizeof(R) / 4;
  uint32_t w[NWD];
#pragma unroll
  for (int i = 0; i < NR; ++i) {
    if constexpr (sizeof(R) == 8) {
      const unsigned long long b = (unsigned long long)__double_as_longlong((double)x[i]);
      w[2 * i] = (uint32_t)b;
      w[2 * i + 1] = (uint32_t)(b >> 32);
    } else {
      w[i] = __float_as_uint((float)x[i]);
    }
  }
  static_assert(NWD % 8 == 0, "TMEM chunks of 8 columns");
  static_for<0, NWD, 8>([&](auto c) {
    constexpr int c0 = decltype(c)::value;
    // x16 chunks where 16 columns remain, the tail (if any) as x8; c0 = 16 j + 8 is covered by the x16 at 16 j
    if constexpr (c0 % 16 == 0 && c0 + 16 <= NWD) tm_st<16>(taddr + col0 + c0, w + c0);
    else if constexpr (!(c0 % 16 == 8 && c0 + 8 <= NWD)) tm_st<8>(taddr + col0 + c0, w + c0);
  });
}
template <typename R, int NR>
__device__ __forceinline__ void tm_load_reals(uint32_t taddr, int col0, R* x) {
  constexpr int NWD = NR * (int)sizeof(R) / 4;
  uint32_t w[NWD];
  static_for<0, NWD, 8>([&](auto c) {
    constexpr int c0 = decltype(c)::value;
    // x16 chunks where 16 columns remain, the tail (if any) as x8; c0 = 16 j + 8 is covered by the x16 at 16 j
    if constexpr (c0 % 16 == 0 && c0 + 16 <= NWD) tm_ld<16>(taddr + col0 + c0, w + c0);
    else if constexpr (!(c0 % 16 == 8 && c0 + 8 <= NWD)) tm_ld<8>(taddr + col0 + c0, w + c0);
  });
  tm_wait_ld();
#pragma unroll
  for (int i = 0; i < NR; ++i) {
    if constexpr (sizeof(R) == 8) {
      x[i] = (R)__longlong_as_double((long long)(((unsigned long long)w[2 * i + 1] << 32) | w[2 * i]));
    } else {
      x[i] = (R)__uint_as_float(w[i]);
    }
  }
}

// dst[i] = sum_j src[off_j(i)] (4 terms) for the ET elements of the group.  The thread's
// outputs i = q + TG k are fully unrolled; table loads use a clamped index so they can all be
// issued before the shared-memory gathers (ILP), only the stores are predicated.
#if BBW_RED32
using red_entry = uint32_t;  // packed RED entry (layout.hpp): offset of b+e0 | delta(b+e2) << 16 | delta(b+e3) << 24
#else
using red_entry = ushort4;
#endif
template <class C, typename R, int CNT, int SRC, int DST, bool DEFER = C::DEFER>
__device__ __forceinline__ void sum4_phase(char* gb, int q, const red_entry* __restrict__ tab) {
  constexpr int K = (CNT + C::TG - 1) / C::TG;
  red_entry o[K];
  R v[K][C::ET];
#pragma unroll
  for (int k = 0; k < K; ++k) o[k] = __ldg(tab + cmin(q + C::TG * k, CNT - 1));
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int i = q + C::TG * k;
    (void)i;
#if BBW_RED32
    const char* p0 = gb + (o[k] & 0xFFFFu) + SRC * C::RB;
    const char* p1 = p0 + C::RB;
    const char* p2 = p0 + ((o[k] >> 16) & 0xFFu) * C::RB;
    const char* p3 = p0 + (o[k] >> 24) * C::RB;
#else
    const char* p0 = gb + o[k].x + SRC * C::RB;
    const char* p1 = gb + o[k].y + SRC * C::RB;
    const char* p2 = gb + o[k].z + SRC * C::RB;
    const char* p3 = gb + o[k].w + SRC * C::RB;
#endif
#pragma unroll
    for (int u = 0; u < C::ET; ++u)
      v[k][u] = (ld<R>(p0 + u * C::EB) + ld<R>(p1 + u * C::EB)) + (ld<R>(p2 + u * C::EB) + ld<R>(p3 + u * C::EB));
    if (!DEFER && ((CNT % C::TG == 0) || i < CNT)) {
#pragma unroll
      for (int u = 0; u < C::ET; ++u) st<R>(gb + DST * C::RB + u * C::EB + i * C::RB, v[k][u]);
    }
  }
  if constexpr (DEFER) {
    // stores after all loads: a store between two outputs' loads would order them (the compiler cannot prove
    // SRC and DST disjoint), serialising one shared-memory round trip per output
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int i = q + C::TG * k;
      if ((CNT % C::TG == 0) || i < CNT) {
#pragma unroll
        for (int u = 0; u < C::ET; ++u) st<R>(gb + DST * C::RB + u * C::EB + i * C::RB, v[k][u]);
      }
    }
  }
}

// dst_ff[i] = scale(i) * sum_s src_ff[off_s(i)] (3 terms) for the 8 face/flux arrays, ET elements.
// Small triangles (the top lift layers) split the 8 arrays over NG lane groups (NG * CNT <= 32), so a
// warp issues 24/NG instead of 24 loads for them; each lane still loads its table entry once.
template <class C, typename R, int CNT, int SRC, int SSTRIDE, int DST, int DSTRIDE, bool SCALED, int SNUM = 1,
          int SDEN = 1>
__device__ __forceinline__ void face_sum3(char* gb, int q, const ushort4* __restrict__ tab, const R* __restrict__ scale) {
  constexpr double MU = double(SNUM) / double(SDEN);  // constant factor of every output (lift layers)
  constexpr int NG = C::TG != 32 ? 1 : (8 * CNT <= 32) ? 8 : (4 * CNT <= 32) ? 4 : (2 * CNT <= 32) ? 2 : 1;  // (-3 % at TG=64)
  constexpr int GF = 8 / NG;  // arrays per lane
  if constexpr (NG == 1) {
    constexpr int K = (CNT + C::TG - 1) / C::TG;
    ushort4 o[K];
    R sc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int ic = cmin(q + C::TG * k, CNT - 1);
      o[k] = __ldg(tab + ic);
      sc[k] = SCALED ? __ldg(scale + ic) : R(1);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int i = q + C::TG * k;
      if (!((CNT % C::TG == 0) || i < CNT)) continue;
      const char* p0 = gb + o[k].x + SRC * C::RB;
      const char* p1 = gb + o[k].y + SRC * C::RB;
      const char* p2 = gb + o[k].z + SRC * C::RB;
      R vv[8][C::ET];
#pragma unroll
      for (int ff = 0; ff < 8; ++ff)
#pragma unroll
        for (int u = 0; u < C::ET; ++u) {
          const int so = ff * SSTRIDE * C::RB + u * C::EB;
          R v = ld<R>(p0 + so) + ld<R>(p1 + so) + ld<R>(p2 + so);
          if constexpr (SCALED) v *= sc[k];
          if constexpr (SNUM != SDEN) v *= R(MU);
          vv[ff][u] = v;
          if constexpr (!C::DEFER) st<R>(gb + (DST + ff * DSTRIDE + i) * C::RB + u * C::EB, v);
        }
      if constexpr (C::DEFER) {  // the 8 arrays' stores after their loads (see sum4_phase)
#pragma unroll
        for (int ff = 0; ff < 8; ++ff)
#pragma unroll
          for (int u = 0; u < C::ET; ++u) st<R>(gb + (DST + ff * DSTRIDE + i) * C::RB + u * C::EB, vv[ff][u]);
      }
    }
  } else {
    if (q < NG * CNT) {
      const int g = q / CNT, i = q - g * CNT;
      const ushort4 o = __ldg(tab + i);
      const R sc = SCALED ? __ldg(scale + i) : R(1);
      const int fo = g * GF * SSTRIDE * C::RB;
      const char* p0 = gb + o.x + SRC * C::RB + fo;
      const char* p1 = gb + o.y + SRC * C::RB + fo;
      const char* p2 = gb + o.z + SRC * C::RB + fo;
      char* d = gb + (DST + g * GF * DSTRIDE + i) * C::RB;
      R vv[GF][C::ET];
#pragma unroll
      for (int ff = 0; ff < GF; ++ff)
#pragma unroll
        for (int u = 0; u < C::ET; ++u) {
          const int so = ff * SSTRIDE * C::RB + u * C::EB;
          R v = ld<R>(p0 + so) + ld<R>(p1 + so) + ld<R>(p2 + so);
          if constexpr (SCALED) v *= sc;
          if constexpr (SNUM != SDEN) v *= R(MU);
          vv[ff][u] = v;
          if constexpr (!C::DEFER) st<R>(d + ff * DSTRIDE * C::RB + u * C::EB, v);
        }
      if constexpr (C::DEFER) {
#pragma unroll
        for (int ff = 0; ff < GF; ++ff)
#pragma unroll
          for (int u = 0; u < C::ET; ++u) st<R>(d + ff * DSTRIDE * C::RB + u * C::EB, vv[ff][u]);
      }
    }
  }
}

// zero reals [off, off + cnt) of every element of the group with 16-B stores (off, cnt multiples of VEC)
template <class C>
__device__ __forceinline__ void zero_region(char* gb, int q, int off, int cnt) {
  const int nv = cnt / C::VEC;
  for (int t = q; t < C::ET * nv; t += C::TG) {
    const int u = t / nv, w = t - u * nv;
    *reinterpret_cast<uint4*>(gb + u * C::EB + off * C::RB + 16 * w) = make_uint4(0, 0, 0, 0);
  }
}

// 1/((m)!)^2 for a runtime m known to lie in [LO, HI] (select chain over compile-time constants)
template <typename R, int LO, int HI>
__device__ __forceinline__ R inv_fact2_sel(int m) {
  R r = R(1.0 / fact2c(LO > 0 ? LO : 0));
  static_for<LO + 1, HI + 1, 1>([&](auto mc) {
    constexpr int mm = decltype(mc)::value;
    if (m == mm) r = R(1.0 / fact2c(mm));
  });
  return r;
}

// G, H, I of the telescoping projection (Eq. telescope) with SHELL-ORDER ownership
// (layout.hpp): lane q owns the multi-indices t with shell index f = q + TG k at every degree, keeps its
// own value of the current level in a register (the e_0 term of every one-degree reduction/elevation),
// and reads only the three other stencil operands from shared memory, at offsets that are the same for
// every degree (SHD/SHU, loaded once per element); outputs are stored at f (contiguous, conflict-free).
//   G/H: u_{n-1}[t] = u_n[t] + u_n[t+e1] + u_n[t+e2] + u_n[t+e3]          (factorial-scaled)
//   I:   b_n[t]   = b_{n-1}[t] + sum_j b_{n-1}[t-e_j] + gam_n u_n[t] / (a!)^2,   b_0 = gam_0 u_0
// On return ob[k] holds b_N at f = q + TG k (k < KO).
template <class C, typename R>
__device__ __forceinline__ void tri_projection(char* gb, int q, const StageArgs<R>& A, const GroupSync<C>& sync,
                                               long long& pt_prev, R* ob) {
  constexpr int N = C::N, M = C::M, NP = C::NP, RB = C::RB, TG = C::TG, KO = C::KO;
  constexpr TabLayout L = tab_layout(N, M, RB);
  const uint8_t* tab = A.tab;
  constexpr int NOUT0 = cnp3(cmax(N + M - 1, N - 1));
  constexpr int KD = (NOUT0 + TG - 1) / TG;
  const uint32_t* shd = reinterpret_cast<const uint32_t*>(tab + L.shd);
  uint32_t sd[KD];
#pragma unroll
  for (int k = 0; k < KD; ++k) sd[k] = __ldg(shd + cmin(q + TG * k, NOUT0 - 1));
  R own[KD];
  // one-degree reduction of the level at SRC (degree n) into DST (degree n-1), own values in registers
  auto reduce = [&](auto srcc, auto dstc, auto nc, auto firstc) {
    constexpr int SRC = decltype(srcc)::value, DST = decltype(dstc)::value, n = decltype(nc)::value;
    constexpr bool FIRST = decltype(firstc)::value;
    constexpr int NOUT = cnp3(n - 1), K = (NOUT + TG - 1) / TG;
    static_for<0, K, 1>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      const int f = q + TG * k;
      if ((NOUT % TG == 0 && k < K) || f < NOUT) {
        const int f1 = (int)(sd[k] & 0xFFFF), de = (int)(sd[k] >> 16);
        const char* sp = gb + (SRC + f1) * RB;
        if constexpr (FIRST) own[k] = ld<R>(gb + (SRC + f) * RB);
        const R v = (own[k] + ld<R>(sp)) + (ld<R>(sp + RB) + ld<R>(sp + de * RB));
        st<R>(gb + (DST + f) * RB, v);
        own[k] = v;
      }
    });
  };
  // G: M reductions N+M -> N (ping-pong T_H <-> T_P; the last lands in level N)
  static_for<N + M, N, -1>([&](auto nc) {
    constexpr int n = decltype(nc)::value;
    constexpr int k = N + M - n;
    constexpr int SRC = (k % 2 == 0) ? C::T_H : C::T_P;
    constexpr int DST = (n - 1 == N) ? C::tlev(N) : ((k % 2 == 0) ? C::T_P : C::T_H);
    reduce(std::integral_constant<int, SRC>{}, std::integral_constant<int, DST>{}, nc,
           std::integral_constant<bool, k == 0>{});
    sync();
    BBW_PT(7);
  });
  // zero slots in front of levels 0..N-1, read by the upward sweep for missing t - e_j (after G: the
  // level region may alias the G buffers)
  if (q < N) st<R>(gb + (C::tlev(q) - 1) * RB, R(0));
  // H: downward reductions level n -> n-1 (levels kept for I)
  static_for<N, 0, -1>([&](auto nc) {
    constexpr int n = decltype(nc)::value;
    reduce(std::integral_constant<int, C::tlev(n)>{}, std::integral_constant<int, C::tlev(n - 1)>{}, nc,
           std::integral_constant<bool, M == 0 && n == N>{});
    sync();
    BBW_PT(8);
  });
  // I: upward, in place (b_n overwrites u_n)
  const uint32_t* shu = reinterpret_cast<const uint32_t*>(tab + L.shu);
  const R* shw = reinterpret_cast<const R*>(tab + L.shw);
  uint32_t su[KO];
  R wk[KO];
#pragma unroll
  for (int k = 0; k < KO; ++k) {
    const int fc = cmin(q + TG * k, NP - 1);
    su[k] = __ldg(shu + fc);
    wk[k] = __ldg(shw + fc);
  }
  if (q == 0) {
    const R b0 = A.gam[0] * ld<R>(gb + C::tlev(0) * RB);
    st<R>(gb + C::tlev(0) * RB, b0);
    ob[0] = b0;
  }
  sync();
  static_for<1, N + 1, 1>([&](auto nc) {
    constexpr int n = decltype(nc)::value;
    constexpr int NOUT = cnp3(n), NPREV = cnp3(n - 1), K = (NOUT + TG - 1) / TG;
    constexpr int BP = C::tlev(n - 1) - 1;  // zero slot of level n-1; SHU offsets are f + 1
    const R gn = A.gam[n];
    static_for<0, K, 1>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      const int f = q + TG * k;
      if ((NOUT % TG == 0 && k < K) || f < NOUT) {
        constexpr int DLO = shell_of(TG * k), DHI = shell_of(cmin(TG * k + TG, NOUT) - 1);
        const uint32_t u = su[k];
        const int d = (int)(u >> 24);
        const R w = gn * wk[k] * inv_fact2_sel<R, n - DHI, n - DLO>(n - d);
        const R un = ld<R>(gb + (C::tlev(n) + f) * RB);
        R v = (ld<R>(gb + (BP + (int)(u & 0xFF)) * RB) + ld<R>(gb + (BP + (int)((u >> 8) & 0xFF)) * RB)) +
              ld<R>(gb + (BP + (int)((u >> 16) & 0xFF)) * RB);
        if constexpr (k * TG < NPREV) {
          if (f < NPREV) v += ob[k];
        }
        v = fma(w, un, v);
        st<R>(gb + (C::tlev(n) + f) * RB, v);
        ob[k] = v;
      }
    });
    sync();
    BBW_PT(9);
  });
}

template <class C, typename R, bool DEFER = C::DEFER>
__device__ __forceinline__ void wadg_phases(char* gb, int q, const StageArgs<R>& A, const GroupSync<C>& sync,
                                            long long& pt_prev, R* ob) {
  R* osc = ob;  // v4 path: output scales of J
  constexpr int N = C::N, M = C::M, NP = C::NP, NPH = C::NPH, RB = C::RB, ET = C::ET, EB = C::EB, TG = C::TG;
  (void)NPH;
  constexpr TabLayout L = tab_layout(N, M, RB);
  const uint8_t* tab = A.tab;
  const R* post = reinterpret_cast<const R*>(tab + L.s_post);
  const R* rowpost = reinterpret_cast<const R*>(tab + L.s_rowpost);
  const red_entry* red = reinterpret_cast<const red_entry*>(tab + L.red);

#if BBW_PROD_V5
  // F (v5): h'_g = post_g * sum_{a+b=g} r''_a c''_b (Eq. mcoeff), output-row stationary with
  // the c''-row loop OUTSIDE the warp passes: every c''-row (b2,b3) is loaded once per element (not once
  // per pass), and each lane loads only the vectors of ITS input row (g2-b2, g3-b3) that exist
  // (predicated on the lane's own row length, not on the warp's longest row), so shared-memory bytes
  // follow the real rows; the FMAs of a vector run under the same predicate.  All passes' row
  // accumulators are live at once; pass k only holds rows with g2+g3 >= SMIN(k) (ROWDEC is sorted by
  // g2+g3 and permuted only within 32-row blocks), which bounds its compile-time row length.
  {
    static_assert(ET == 1, "product v5 assumes one element per group batch");
    constexpr int NR = cnp2(N + M), KR = (NR + TG - 1) / TG;
    constexpr int VEC = C::VEC, RS = C::RS, LH = N + M + 1;
    const uint32_t* rowdec = reinterpret_cast<const uint32_t*>(tab + L.rowdec);
    int g2v[KR], g3v[KR], gsv[KR], rid0v[KR];
    bool actv[KR];
    R rowfv[KR];
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int rho = q + TG * k;
      actv[k] = rho < NR;
      const uint32_t d = __ldg(rowdec + (actv[k] ? rho : NR - 1));
      rowfv[k] = __ldg(rowpost + (actv[k] ? rho : NR - 1));
      g2v[k] = d & 0xFF;
      g3v[k] = (d >> 8) & 0xFF;
      gsv[k] = (int)(d >> 16);
      rid0v[k] = g3v[k] * (2 * N + 3 - g3v[k]) / 2 + g2v[k];
    }
    // flat accumulator: pass k owns entries [AOFF(k), AOFF(k) + LH - SMIN(k)) (compile-time sizes)
    constexpr int ATOT = prod_acc_total(N + M, TG, KR);
    R acc[ET][ATOT];
#pragma unroll
    for (int u = 0; u < ET; ++u)
#pragma unroll
      for (int x = 0; x < ATOT; ++x) acc[u][x] = R(0);
    static_for<0, M + 1, 1>([&](auto b3c) {
      constexpr int b3 = decltype(b3c)::value;
      static_for<0, M + 1 - b3, 1>([&](auto b2c) {
        constexpr int b2 = decltype(b2c)::value;
        constexpr int LB = M - b2 - b3 + 1;
        constexpr int CB = cnp3(M) - cnp3(M - b3) + b2 * (2 * (M - b3) + 3 - b2) / 2;  // rank_M(0,b2,b3)
        R cv[ET][LB];
#pragma unroll
        for (int u = 0; u < ET; ++u)
#pragma unroll
          for (int b1 = 0; b1 < LB; ++b1) cv[u][b1] = ld<R>(gb + (C::O_C + CB + b1) * RB + u * EB);
        static_for<0, KR, 1>([&](auto kc) {
          constexpr int k = decltype(kc)::value;
          constexpr int SMIN = prod_pass_smin(TG * k);
          constexpr int LA = cmin(N + 1, N + 1 - SMIN + b2 + b3);  // longest input row pass k can meet
          if constexpr (LA > 0) {
            const int a2 = g2v[k] - b2, a3 = g3v[k] - b3;
            const bool valid = actv[k] && a2 >= 0 && a3 >= 0 && a2 + a3 <= N;
            const int lenA = valid ? N + 1 - a2 - a3 : 0;
            const int lamax = __reduce_max_sync(0xffffffffu, lenA);
            if (lamax > 0) {
              const int rid = rid0v[k] + b3 * g3v[k] - b3 * (2 * N + 3 + b3) / 2 - b2;  // rowid(a2, a3)
              const char* pr = gb + (C::Y_RPP + (valid ? rid : 0) * RS) * RB;
#pragma unroll
              for (int u = 0; u < ET; ++u) {
                const unsigned pa = (unsigned)__cvta_generic_to_shared(pr + u * EB);
                static_for<0, LA, VEC>([&](auto vc) {
                  constexpr int v0 = decltype(vc)::value;
                  if (v0 < lamax) {  // warp-uniform
                    const bool pv = v0 < lenA;
                    R x[VEC];
#pragma unroll
                    for (int i = 0; i < VEC; ++i) x[i] = R(0);
                    ld_shared_vec_pred<R, v0 * C::RB>(x, pa, pv);
#pragma unroll
                    for (int i = 0; i < VEC; ++i) {
                      if (v0 + i < LA) {
#pragma unroll
                        for (int b1 = 0; b1 < LB; ++b1) {
                          constexpr int AO = prod_acc_off(N + M, TG, k);
                          acc[u][AO + v0 + i + b1] = fma(cv[u][b1], x[i], acc[u][AO + v0 + i + b1]);
                        }
                      }
                    }
                  }
                });
              }
            }
          }
        });
      });
    });
    // outputs: h'_g = N!M!/(N+M)! (g!)^2 h''_g, g = (lg-1-x, x, g2, g3), as v4 below
    static_for<0, KR, 1>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      constexpr int LMAX = LH - prod_pass_smin(TG * k);
      constexpr int AO = prod_acc_off(N + M, TG, k);
      if (actv[k]) {
        const int lg = N + M - g2v[k] - g3v[k] + 1;
        // TRIPLE: shell index of t = (x, g2, g3): f = Np(d-1) + g3 (2d+3-g3)/2 + g2, d = x + g2 + g3, stepped
        // down in x; otherwise the canonical degree-(N+M) rank gs + x
        constexpr int DSTH = (M == 0) ? C::tlev(N) : C::T_H;
        const int sg = g2v[k] + g3v[k];
        int dd = LMAX - 1 + sg;
        int fx = dd * (dd + 1) * (dd + 2) / 6 + g3v[k] * (2 * dd + 3 - g3v[k]) / 2 + g2v[k];
        int Dn = dd * (dd + 1) / 2;  // Nfp(d-1)
        (void)DSTH;
        (void)fx;
        (void)Dn;
#define BBW_HSTORE(xx, val)                                        \
  do {                                                             \
    if constexpr (C::TRIPLE) st<R>(gb + (DSTH + fx) * RB, (val));   \
    else st<R>(gb + (C::W_H + gsv[k] + (xx)) * RB, (val));         \
  } while (0)
#define BBW_HSTEP()                \
  do {                             \
    if constexpr (C::TRIPLE) {     \
      fx -= Dn + g3v[k];           \
      Dn -= dd;                    \
      --dd;                        \
    }                              \
  } while (0)
        if constexpr (N + M <= 12) {
          R P = rowfv[k], T = R(lg - (N + M));
          static_for<N + M, -1, -1>([&](auto xc) {
            constexpr int x = decltype(xc)::value;
            if constexpr (x < LMAX) {
              if (x < lg) BBW_HSTORE(x, acc[0][AO + x] * (R(fact2c(x)) * P));
              if constexpr (x > 0) BBW_HSTEP();
            }
            const R Tc = T > R(1) ? T : R(1);
            P *= Tc * Tc;
            T += R(1);
          });
        } else {
          static_for<LMAX - 1, -1, -1>([&](auto xc) {
            constexpr int x = decltype(xc)::value;
            if (x < lg) BBW_HSTORE(x, acc[0][AO + x] * __ldg(post + gsv[k] + x));
            if constexpr (x > 0) BBW_HSTEP();
          });
        }
#undef BBW_HSTORE
#undef BBW_HSTEP
      }
    });
  }
#else
  // F: h'_g = post_g * sum_{a+b=g} r''_a c''_b, output-row stationary: for output row (g2,g3) of
  // degree N+M and every c''-row (b2,b3), the input row (g2-b2, g3-b3) of r'' is loaded once into
  // registers and convolved (1-D, full) with the c''-row into the row accumulators.
  {
    constexpr int NR = cnp2(N + M), KR = (NR + TG - 1) / TG;
    const uint32_t* rowdec = reinterpret_cast<const uint32_t*>(tab + L.rowdec);
    // Rows are stored in order of increasing g2 + g3 (tables.cpp), so the rows of one warp pass
    // have similar lengths.  r'' is read from its zero-padded row copy (16-B vector loads; lanes
    // whose input row does not exist read the zero row), and the unrolled a1 steps beyond the
    // warp's longest input row (la_max = N+1 - (min g2+g3 over the warp) + b2 + b3) are skipped by
    // warp-uniform branches, so the FMA count follows the real row lengths.
    constexpr int VEC = C::VEC, RS = C::RS;
    R x[RS + VEC];
#pragma unroll
    for (int i = 0; i < RS + VEC; ++i) x[i] = R(0);
#pragma unroll 1
    for (int k = 0; k < KR; ++k) {
      const int rho = q + TG * k;
      const bool act = rho < NR;
      const uint32_t d = __ldg(rowdec + (act ? rho : NR - 1));
      const R rowf = __ldg(rowpost + (act ? rho : NR - 1));
      const int g2 = d & 0xFF, g3 = (d >> 8) & 0xFF, gs = (int)(d >> 16);
      const int smin = __reduce_min_sync(0xffffffffu, act ? g2 + g3 : 4 * (N + M));
      // rowid(a2, a3) = a3 (2N+3-a3)/2 + a2 at a = G - B: rid0 + b3 g3 - b3 (2N+3+b3)/2 - b2
      const int rid0 = g3 * (2 * N + 3 - g3) / 2 + g2;
      R acc[ET][N + M + 1];
#pragma unroll
      for (int u = 0; u < ET; ++u)
#pragma unroll
        for (int x = 0; x <= N + M; ++x) acc[u][x] = R(0);
      static_for<0, M + 1, 1>([&](auto b3c) {
        constexpr int b3 = decltype(b3c)::value;
        const int rid3 = rid0 + b3 * g3 - b3 * (2 * N + 3 + b3) / 2;
        static_for<0, M + 1 - b3, 1>([&](auto b2c) {
          constexpr int b2 = decltype(b2c)::value;
          constexpr int LB = M - b2 - b3 + 1;
          constexpr int CB = cnp3(M) - cnp3(M - b3) + b2 * (2 * (M - b3) + 3 - b2) / 2;  // rank_M(0,b2,b3)
          const int a2 = g2 - b2, a3 = g3 - b3;
          const bool valid = act && a2 >= 0 && a3 >= 0 && a2 + a3 <= N;
          if (__any_sync(0xffffffffu, valid)) {
            const int lamax = cmin(N + 1, N + 1 - smin + b2 + b3);
            const char* pr = gb + (C::Y_RPP + (valid ? rid3 - b2 : C::NFP) * RS) * RB;
#pragma unroll
            for (int u = 0; u < ET; ++u) {
              R cv[LB];
#pragma unroll
              for (int b1 = 0; b1 < LB; ++b1) cv[b1] = ld<R>(gb + (C::O_C + CB + b1) * RB + u * EB);
              // only the vectors below the warp's la_max are loaded and only the a1 < la_max FMAs run:
              // warp-uniform jumps into fall-through sequences (x keeps stale values above la_max,
              // which are never read; the loads are opaque asm so x stays in registers)
              const unsigned pa = (unsigned)__cvta_generic_to_shared(pr + u * EB);
#if BBW_PROD_SWITCH
              auto ldv = [&](auto vc) {
                constexpr int a1 = decltype(vc)::value * VEC;
                if constexpr (a1 <= N) ld_shared_vec<R, a1 * C::RB>(&x[a1], pa);
              };
              BBW_FALLTHROUGH_SWITCH((lamax + VEC - 1) / VEC, ldv);
              auto fm = [&](auto a1c) {
                constexpr int a1 = decltype(a1c)::value;
                if constexpr (a1 <= N) {
#pragma unroll
                  for (int b1 = 0; b1 < LB; ++b1) acc[u][a1 + b1] = fma(cv[b1], x[a1], acc[u][a1 + b1]);
                }
              };
              BBW_FALLTHROUGH_SWITCH(lamax, fm);
#else
              static_for<0, N + 1, VEC>([&](auto a1c) {
                constexpr int a1 = decltype(a1c)::value;
                ld_shared_vec_pred<R, a1 * C::RB>(&x[a1], pa, a1 < lamax);
              });
              static_for<0, N + 1, 1>([&](auto a1c) {
                constexpr int a1 = decltype(a1c)::value;
                if (a1 < lamax) {
#pragma unroll
                  for (int b1 = 0; b1 < LB; ++b1) acc[u][a1 + b1] = fma(cv[b1], x[a1], acc[u][a1 + b1]);
                }
              });
#endif
            }
          }
        });
      });
      if (act) {
        // h'_g = N!M!/(N+M)! (g!)^2 h''_g with g = (lg-1-x, x, g2, g3): the row factor comes from
        // ROWPOST, (x!)^2 is a compile-time constant and (g0!)^2 a running product over x = lg-1 .. 0
        // (no per-output table load)
        const int lg = N + M - g2 - g3 + 1;
        if constexpr (N + M <= 12) {
          R P = rowf, T = R(lg - (N + M));
          static_for<N + M, -1, -1>([&](auto xc) {
            constexpr int x = decltype(xc)::value;
            if (x < lg) {
#pragma unroll
              for (int u = 0; u < ET; ++u)
                st<R>(gb + (C::W_H + gs + x) * RB + u * EB, acc[u][x] * (R(fact2c(x)) * P));
            }
            const R Tc = T > R(1) ? T : R(1);  // (g0 + 1)^2 for x < lg, 1 above the row
            P *= Tc * Tc;
            T += R(1);
          });
        } else {  // long rows (N+M > 12): the per-output table is faster (measured at N = M = 9)
#pragma unroll
          for (int x = 0; x <= N + M; ++x) {
            if (x < lg) {
              const R sp = __ldg(post + gs + x);
#pragma unroll
              for (int u = 0; u < ET; ++u) st<R>(gb + (C::W_H + gs + x) * RB + u * EB, acc[u][x] * sp);
            }
          }
        }
      }
    }
  }
#endif
  sync();
  BBW_PT(6);
  if constexpr (C::TRIPLE) {
    tri_projection<C, R>(gb, q, A, sync, pt_prev, ob);
    return;
  }
  if constexpr (!C::ALIAS) {
    if (q == 0) {  // zero slots of the upward-sweep ping-pong buffers (may alias the padded rows read above)
#pragma unroll
      for (int u = 0; u < ET; ++u) {
        st<R>(gb + C::W_A0 * RB + u * EB, R(0));
        st<R>(gb + C::W_A1 * RB + u * EB, R(0));
      }
    }
  }
  // the output scales a!/N! of phase J are requested here, off its critical path
  {
    const R* outN = reinterpret_cast<const R*>(tab + L.s_outN);
#pragma unroll
    for (int k = 0; k < C::KO; ++k) osc[k] = __ldg(outN + cmin(q + TG * k, NP - 1));
  }
  // G: M reductions N+M -> N (ping-pong H <-> P; the last lands in level N)
  static_for<N + M, N, -1>([&](auto nc) {
    constexpr int n = decltype(nc)::value;
    constexpr int k = N + M - n;
    constexpr int SRC = (k % 2 == 0) ? C::W_H : C::W_P;
    constexpr int DST = (n - 1 == N) ? C::lev(N) : ((k % 2 == 0) ? C::W_P : C::W_H);
    sum4_phase<C, R, cnp3(n - 1), SRC, DST, DEFER>(gb, q, red + red_off(n));
    sync();
    BBW_PT(7);
  });
  if constexpr (M == 0) {
    for (int i = q; i < NP; i += TG)
#pragma unroll
      for (int u = 0; u < ET; ++u)
        st<R>(gb + (C::lev(N) + i) * RB + u * EB, ld<R>(gb + (C::W_H + i) * RB + u * EB));
    sync();
    BBW_PT(7);
  }
  // zero slots read by the upward sweep in front of levels 0..N-1 (ALIAS: the region held h / P until now)
  if constexpr (C::ALIAS) {
    if (q < N) {
#pragma unroll
      for (int u = 0; u < ET; ++u) st<R>(gb + (C::lev(q) - 1) * RB + u * EB, R(0));
    }
  }
  // H: downward reductions level n -> n-1
  static_for<N, 0, -1>([&](auto nc) {
    constexpr int n = decltype(nc)::value;
    sum4_phase<C, R, cnp3(n - 1), C::lev(n), C::lev(n - 1), DEFER>(gb, q, red + red_off(n));
    sync();
    BBW_PT(8);
  });
  // I: upward, in place: b_n[a] = sum_j b_{n-1}[a - e_j] + gam_n/(a!)^2 u_n[a] overwrites u_n (b_0 = gam_0 u_0)
  static_for<1, N + 1, 1>([&](auto nc) {
    constexpr int n = decltype(nc)::value;
    // UPW offsets are (rank + 1) * RB, 0 = the zero slot; b_n -> level n in place (ALIAS) or A_{n%2}
    constexpr int SRC = C::ALIAS ? C::lev(n - 1) - 1 : ((n % 2 == 1) ? C::W_A0 : C::W_A1);
    constexpr int DST = C::ALIAS ? C::lev(n) : ((n % 2 == 1) ? C::W_A1 : C::W_A0) + 1;
    const R gn = A.gam[n];
    if constexpr (n == 1) {
      // degree 1: every a has exactly one valid a - e_j (= the single b_0), weight 1/(a!)^2 = 1
      const R g0 = A.gam[0];
      for (int i = q; i < 4; i += TG)
#pragma unroll
        for (int u = 0; u < ET; ++u) {
          const R b0 = g0 * ld<R>(gb + C::lev(0) * RB + u * EB);
          st<R>(gb + (DST + i) * RB + u * EB, fma(gn, ld<R>(gb + (C::lev(1) + i) * RB + u * EB), b0));
        }
    } else {
      const uint8_t* up = tab + L.upw + 16 * upw_off(n);
      constexpr int CNT = cnp3(n), K = (CNT + TG - 1) / TG;
      ushort4 o[K];
      R w[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int ic = cmin(q + TG * k, CNT - 1);
        o[k] = __ldg(reinterpret_cast<const ushort4*>(up + 16 * ic));
        w[k] = gn * __ldg(reinterpret_cast<const R*>(up + 16 * ic + 8));
      }
      R v[K][ET];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int i = q + TG * k;
        const char* p0 = gb + o[k].x + SRC * RB;
        const char* p1 = gb + o[k].y + SRC * RB;
        const char* p2 = gb + o[k].z + SRC * RB;
        const char* p3 = gb + o[k].w + SRC * RB;
#pragma unroll
        for (int u = 0; u < ET; ++u) {
          v[k][u] = (ld<R>(p0 + u * EB) + ld<R>(p1 + u * EB)) + (ld<R>(p2 + u * EB) + ld<R>(p3 + u * EB));
          v[k][u] = fma(w[k], ld<R>(gb + (C::lev(n) + cmin(i, CNT - 1)) * RB + u * EB), v[k][u]);
        }
        if (!DEFER && ((CNT % TG == 0) || i < CNT)) {
#pragma unroll
          for (int u = 0; u < ET; ++u) st<R>(gb + (DST + i) * RB + u * EB, v[k][u]);
        }
      }
      if constexpr (DEFER) {  // in place: lane-private u_n[i] is read above before its own store here
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int i = q + TG * k;
          if ((CNT % TG == 0) || i < CNT) {
#pragma unroll
            for (int u = 0; u < ET; ++u) st<R>(gb + (DST + i) * RB + u * EB, v[k][u]);
          }
        }
      }
    }
    sync();
    BBW_PT(9);
  });
}

template <class C>
__host__ __device__ constexpr int wadg_result() {
  return C::ALIAS ? C::lev(C::N) : ((C::N % 2 == 1) ? C::W_A1 + 1 : C::W_A0 + 1);
}

template <class C, typename R>
__global__ void __launch_bounds__(C::T, C::MINB) stage_kernel(const StageArgs<R> A) {
  constexpr int N = C::N, M = C::M, NP = C::NP, NFP = C::NFP, NFP1 = C::NFP1, MP = C::MP, NPM1 = C::NPM1;
  constexpr int ET = C::ET, EB = C::EB, RB = C::RB, TG = C::TG, VEC = C::VEC, KO = C::KO;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int grp = tid / TG, q = tid - grp * TG;
  char* gb = reinterpret_cast<char*>(smem_raw) + grp * C::GB;  // this group's elements
  const GroupSync<C> sync{1 + grp};
  constexpr TabLayout L = tab_layout(N, M, RB);
  const uint8_t* tab = A.tab;
  const R* invfacN = reinterpret_cast<const R*>(tab + L.s_invfacN);
  const R* facN = reinterpret_cast<const R*>(tab + L.s_facN);
  const R* outN = reinterpret_cast<const R*>(tab + L.s_outN);
  const R* invfacM = reinterpret_cast<const R*>(tab + L.s_invfacM);
  const R* invfacNm1 = reinterpret_cast<const R*>(tab + L.s_invfacNm1);
  const R* cfac = reinterpret_cast<const R*>(tab + L.s_cfac);
  const uint16_t* fnode = reinterpret_cast<const uint16_t*>(tab + L.fnode);
  const uint16_t* nbrvol = reinterpret_cast<const uint16_t*>(tab + L.nbrvol);
  const uint16_t* nbrface = reinterpret_cast<const uint16_t*>(tab + L.nbrface);

  const long long nelem = A.elem_end - A.elem_begin;
  const long long nbatch = (nelem + ET - 1) / ET;
#define BBW_PA(k) (q + TG * (k))
  // TMA bulk staging for whole-warp groups (N >= 5); the sub-warp groups of N <= 4 stage with cp.async
  // (TMA measured 0 % faster at (7,4); compute-sanitizer racecheck flags the TMA path only for sub-warp groups)
  constexpr bool kTMA = BBW_TMA && BBW_CPASYNC && (TG >= BBW_TMA_MIN_TG);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem_raw + C::G * C::GB) + grp;
  unsigned mbar_phase = 0;
  if constexpr (kTMA) {
    if (q == 0) mbar_init(mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
  }
#if BBW_LSRK_TMEM
  static_assert(ET == 1 && BBW_LSRK_REG, "TMEM LSRK state: one element per batch, register-resident state model");
  // LSRK state columns: residual at [0, TMW), Q_in copy at [TMW, 2 TMW); TMW = 4 KO reals in 32-bit words,
  // rounded up to 8 columns; the allocation (power of 2 >= 32) is per CTA, lanes per warp quadrant
  constexpr int TMR = ((4 * KO * RB / 4 + 7) / 8 * 8) / (RB / 4);  // reals per array, padded
  constexpr int TMW = TMR * RB / 4;
  constexpr int TMCOLS = (2 * TMW <= 32) ? 32 : (2 * TMW <= 64) ? 64 : (2 * TMW <= 128) ? 128 : 256;
  __shared__ uint32_t tmem_base_s;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&tmem_base_s)),
                 "r"(TMCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t taddr = tmem_base_s + ((uint32_t)(32 * ((tid >> 5) & 3)) << 16);
#endif
  // Sub-warp groups (TG < 32) share their warp's synchronisation, so the trip count is uniform per
  // warp: the loop runs over the batch of the warp's first group, idle groups get nE = 0.
  const int gw = grp % C::GPW;
#if BBW_DYNQ
  // Dynamic work queue: each warp (sub-warp groups) or group takes the next GPW batches from a global atomic
  // ticket, so the elements in flight stay a contiguous Morton window even when SMs drift apart over the
  // ~1700 batches per group of a 4M-element launch (a static grid-stride schedule lets the window spread,
  // and the neighbour face traces then miss L2).  The last unit to finish resets the counters, so the next
  // stream-ordered launch (or graph replay) starts from zero.
  auto next_batch = [&]() -> long long {
    if constexpr (TG <= 32) {
      unsigned v = 0;
      if ((tid & 31) == 0) v = atomicAdd(A.qctr, 1u);
      return (long long)__shfl_sync(0xffffffffu, v, 0) * C::GPW;
    } else {
      unsigned* tslot = reinterpret_cast<unsigned*>(smem_raw + C::G * C::GB + 8 * C::G) + grp;
      if (q == 0) *tslot = atomicAdd(A.qctr, 1u);
      sync();
      return (long long)*tslot;
    }
  };
  // A ticket covers QCH consecutive unit-batches: 1 keeps the window tightest (best on the 4M-element config-5
  // mesh), 2 amortises the atomic's L2 round trip on smaller meshes (api.cu picks it; drawing the next ticket at
  // the start of a batch instead measured 2.6 % slower at (7,4)).
  const int QCH = A.qch > 0 ? A.qch : 1;
  long long bw = 0;
  int qleft = 0;
  for (;;) {
    if (qleft == 0) {
      bw = next_batch() * QCH;
      qleft = QCH;
    } else {
      bw += C::GPW;
    }
    --qleft;
    if (bw >= nbatch) break;
#else
  for (long long bw = (long long)blockIdx.x * C::G + (grp - gw); bw < nbatch; bw += (long long)gridDim.x * C::G) {
#endif
    const long long batch = bw + gw;
    const long long k0 = A.elem_begin + batch * ET;
    long long pt_prev = clock64();
    (void)pt_prev;
    // valid elements of the batch (compile-time 1 for ET == 1 and whole-warp groups: every batch
    // start is < elem_end)
    const int nE = (ET == 1 && C::GPW == 1)
                       ? 1
                       : (batch >= nbatch ? 0 : (int)((A.elem_end - k0) < ET ? (A.elem_end - k0) : ET));

    // ---- A: loads (Q, geometry, c'' -> smem via cp.async; the residual is only prefetched into L2
    //      here and read in phases D and J, so no registers are held across the WADG phases)
#if BBW_LSRK_REG
    R rs[ET][4][KO];  // LSRK residual: loaded now, consumed at the end (HBM latency hidden)
    if (A.mode == 0) {
#pragma unroll
      for (int u = 0; u < ET; ++u)
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int k = 0; k < KO; ++k) {
            const int a = c == 0 ? BBW_PA(k) : q + TG * k;
            rs[u][c][k] = (u < nE && q + TG * k < NP) ? __ldcs(A.res + (k0 + u) * 4 * NP + c * NP + a) : R(0);
          }
    }
#else
    if (A.mode == 0) {
      const int nl = (nE * 4 * NP * RB + 127) / 128;
      const char* pr = reinterpret_cast<const char*>(A.res + k0 * 4 * NP);
      for (int l = q; l < nl; l += TG) prefetch_l2(pr + 128 * l);
    }
#endif
    if (A.mode == 2) {
      zero_region<C>(gb, q, C::Y_RPP, C::NS);
      sync();
      const uint16_t* padoff = reinterpret_cast<const uint16_t*>(tab + L.padoff);
      for (int t = q; t < nE * NP; t += TG) {
        const int u = t / NP, a = t - u * NP;
        const R v = A.Qin[(k0 + u) * NP + a] * __ldg(invfacN + a);
        st<R>(gb + u * EB + (C::O_RP + a) * RB, v);
        st<R>(gb + u * EB + C::Y_RPP * RB + __ldg(padoff + a), v);
      }
    } else {
#if BBW_CPASYNC
      // one round trip: every per-element input goes global -> shared with cp.async (LDGSTS)
      constexpr int NV = 4 * NP / VEC;  // 16-B chunks of Q
      constexpr int GV = 12 * RB / 16;  // 16-B chunks of grad(lambda)
      const char* gq = reinterpret_cast<const char*>(A.Qin + k0 * 4 * NP);
      if constexpr (kTMA) {
      // one elected lane per group: Q block (4 Np reals), grad(lambda) (12 reals) and the 4 neighbour ids of
      // every element of the batch by TMA bulk copies on the group's mbarrier (no LSU wavefronts)
      (void)NV;
      (void)gq;
      if (q == 0 && nE > 0) {
        mbar_expect_tx(mbar, (unsigned)nE * (4 * NP * RB + 12 * RB + 16));
        for (int u = 0; u < nE; ++u) {
          char* eb = gb + u * EB;
          bulk_g2s(eb + C::X_Q * RB, A.Qin + (k0 + u) * 4 * NP, 4 * NP * RB, mbar);
          bulk_g2s(eb + C::O_GEO * RB, A.geo + (k0 + u) * 12, 12 * RB, mbar);
          bulk_g2s(eb + 28 * RB, A.nbr + (k0 + u) * 4, 16, mbar);
        }
      }
      for (int u = q; u < nE; u += TG) cp_async4(gb + u * EB + 28 * RB + 16, A.code + (k0 + u) * 4);  // 4 codes
      } else {
#pragma unroll
      for (int t0 = 0; t0 < ET * NV; t0 += TG) {
        const int t = t0 + q;
        if (t < nE * NV) {
          const int u = t / NV, w = t - u * NV;
          cp_async16(gb + u * EB + C::X_Q * RB + w * 16, gq + 16 * t);
        }
      }
      for (int t = q; t < nE * (GV + 2); t += TG) {
        const int u = t / (GV + 2), w = t - u * (GV + 2);
        char* eb = gb + u * EB;
        if (w < GV) cp_async16(eb + C::O_GEO * RB + w * 16, reinterpret_cast<const char*>(A.geo + (k0 + u) * 12) + 16 * w);
        else if (w == GV) cp_async16(eb + 28 * RB, A.nbr + (k0 + u) * 4);     // 4 neighbour ids
        else cp_async4(eb + 28 * RB + 16, A.code + (k0 + u) * 4);             // 4 codes (bytes)
      }
      }
      for (int t = q; t < nE * MP; t += TG) {
        const int u = t / MP, b = t - u * MP;
        cp_async_real<R>(gb + u * EB + (C::O_C + b) * RB, A.c2 + (k0 + u) * MP + b);
      }
#if BBW_PF
      {  // L2 prefetch of the group's next batch (Q_in, residual, c^2)
        const long long kn = A.elem_begin + (batch + (long long)gridDim.x * C::G) * ET;
        if (kn < A.elem_end) {
          const int ne = (int)((A.elem_end - kn) < ET ? (A.elem_end - kn) : ET);
          const int nl = (ne * 4 * NP * RB + 127) / 128;
          const char* pq = reinterpret_cast<const char*>(A.Qin + kn * 4 * NP);
          const char* pr = reinterpret_cast<const char*>(A.res + kn * 4 * NP);
          for (int l = q; l < nl; l += TG) {
            prefetch_l2(pq + 128 * l);
            if (A.mode == 0) prefetch_l2(pr + 128 * l);
          }
          if (q == 0) prefetch_l2(A.c2 + kn * MP);
        }
      }
#endif
      cp_async_wait_all();
      if (kTMA && nE > 0) {
        mbar_wait(mbar, mbar_phase);
        mbar_phase ^= 1;
      }
      sync();
      for (int t = q; t < nE * 4; t += TG) {  // outward normal, |grad lambda_f|
        const int u = t >> 2, f = t & 3;
        char* sg = gb + u * EB + C::O_GEO * RB;
        const R gx = ld<R>(sg + (3 * f) * RB), gy = ld<R>(sg + (3 * f + 1) * RB), gz = ld<R>(sg + (3 * f + 2) * RB);
        const R gl = sqrt(gx * gx + gy * gy + gz * gz), il = R(1) / gl;
        st<R>(sg + (12 + 4 * f) * RB, -gx * il);
        st<R>(sg + (13 + 4 * f) * RB, -gy * il);
        st<R>(sg + (14 + 4 * f) * RB, -gz * il);
        st<R>(sg + (15 + 4 * f) * RB, gl);
      }
      for (int t = q; t < ET * 12; t += TG) {  // zero slots of the G'' (4) and Y'' (8) arrays
        const int u = t / 12, z = t - u * 12;
        const int off = z < 4 ? C::X_G + z * (NPM1 + 1) : C::Y_Y + (z - 4) * (NFP1 + 1);
        st<R>(gb + u * EB + off * RB, R(0));
      }
      for (int t = q; t < nE * MP; t += TG) {  // c'' = c^2 / b!
        const int u = t / MP, b = t - u * MP;
        char* p = gb + u * EB + (C::O_C + b) * RB;
        st<R>(p, ld<R>(p) * __ldg(invfacM + b));
      }
#else
      constexpr int NV = 4 * NP / VEC;
      using V = typename std::conditional<sizeof(R) == 8, double2, float4>::type;
      const V* gq = reinterpret_cast<const V*>(A.Qin + k0 * 4 * NP);
      for (int t = q; t < nE * NV; t += TG) {
        const int u = t / NV, w = t - u * NV;
        *reinterpret_cast<V*>(gb + u * EB + C::X_Q * RB + w * 16) = __ldg(gq + t);
      }
      for (int t = q; t < nE * 4; t += TG) {  // neighbour id and code of every face
        const int u = t >> 2, f = t & 3;
        int* nbs = reinterpret_cast<int*>(gb + u * EB + 28 * RB);
        nbs[f] = __ldg(A.nbr + (k0 + u) * 4 + f);
        reinterpret_cast<uint8_t*>(nbs + 4)[f] = __ldg(A.code + (k0 + u) * 4 + f);
      }
      for (int t = q; t < nE * 4; t += TG) {  // grad lambda_f, outward normal, |grad lambda_f|
        const int u = t >> 2, f = t & 3;
        const R* g = A.geo + (k0 + u) * 12 + 3 * f;
        const R gx = __ldg(g), gy = __ldg(g + 1), gz = __ldg(g + 2);
        const R gl = sqrt(gx * gx + gy * gy + gz * gz), il = R(1) / gl;
        char* sg = gb + u * EB + C::O_GEO * RB;
        st<R>(sg + (3 * f) * RB, gx);
        st<R>(sg + (3 * f + 1) * RB, gy);
        st<R>(sg + (3 * f + 2) * RB, gz);
        st<R>(sg + (12 + 4 * f) * RB, -gx * il);
        st<R>(sg + (13 + 4 * f) * RB, -gy * il);
        st<R>(sg + (14 + 4 * f) * RB, -gz * il);
        st<R>(sg + (15 + 4 * f) * RB, gl);
      }
      for (int t = q; t < ET * 12; t += TG) {  // zero slots of the G'' (4) and Y'' (8) arrays
        const int u = t / 12, z = t - u * 12;
        const int off = z < 4 ? C::X_G + z * (NPM1 + 1) : C::Y_Y + (z - 4) * (NFP1 + 1);
        st<R>(gb + u * EB + off * RB, R(0));
      }
      for (int t = q; t < nE * MP; t += TG) {
        const int u = t / MP, b = t - u * MP;
        st<R>(gb + u * EB + (C::O_C + b) * RB, __ldg(A.c2 + (k0 + u) * MP + b) * __ldg(invfacM + b));
      }
#endif
    }
    if (A.mode == 2) {
      for (int t = q; t < nE * MP; t += TG) {
        const int u = t / MP, b = t - u * MP;
        st<R>(gb + u * EB + (C::O_C + b) * RB, __ldg(A.c2 + (k0 + u) * MP + b) * __ldg(invfacM + b));
      }
    }
    sync();
    BBW_PT(0);

    R ru[ET][3][KO];  // own r_u (x/a! scaled until phase E)
#if BBW_LSRK_REG
    R qo[ET][4][KO];  // own Q_in coefficients (LSRK)
#endif
    if (A.mode != 2) {
      // ---- B1a: neighbour face traces of every flux item are requested first (L2 / DRAM latency),
      //      then B2 runs while they are in flight, then B1b forms the fluxes.
      constexpr int NI1 = 4 * NFP, K1 = (NI1 + TG - 1) / TG;
      R tpp[K1][ET], tux[K1][ET], tuy[K1][ET], tuz[K1][ET];
      int town[K1];
#pragma unroll
      for (int k = 0; k < K1; ++k) {
        const int t = q + TG * k;
        const bool act = (NI1 % TG == 0) || t < NI1;
        const int tc = act ? t : 0;
        const int f = tc / NFP, i = tc - f * NFP;
        town[k] = __ldg(fnode + f * NFP + i);
#pragma unroll
        for (int u = 0; u < ET; ++u) {
          const int* nbs = reinterpret_cast<const int*>(gb + u * EB + 28 * RB);
          const int nb = nbs[f], code = reinterpret_cast<const uint8_t*>(nbs + 4)[f];
          tpp[k][u] = tux[k][u] = tuy[k][u] = tuz[k][u] = R(0);
          if (act && u < nE) {
            if (nb >= 0) {
              const int vol = __ldg(nbrvol + code * NFP + i);
              const R* qn = A.Qin + (long long)nb * 4 * NP + vol;
              tpp[k][u] = __ldg(qn);
              tux[k][u] = __ldg(qn + NP);
              tuy[k][u] = __ldg(qn + 2 * NP);
              tuz[k][u] = __ldg(qn + 3 * NP);
            } else if (nb < -1 && A.gmap) {
              // partition face, peer-read transport: the owner's Q_in, read in place
              const int slot = -2 - nb;
              const int2 gm = __ldg(reinterpret_cast<const int2*>(A.gmap) + slot);
              const int vol = __ldg(nbrvol + code * NFP + i);
              const R* qn = A.peer[gm.x] + (long long)gm.y * 4 * NP + vol;
              tpp[k][u] = __ldg(qn);
              tux[k][u] = __ldg(qn + NP);
              tuy[k][u] = __ldg(qn + 2 * NP);
              tuz[k][u] = __ldg(qn + 3 * NP);
            } else if (nb < -1) {
              // partition face: the halo carries p+ and u+.n+ (n+ = the sender's outward normal = -n);
              // the flux needs only [[p]] and n.[[u]] (Eq. sdf); tux holds u+.n+
              const int fi = __ldg(nbrface + (code % 6) * NFP + i);
              const R* gh = A.ghost + (long long)(-2 - nb) * 2 * NFP + fi;
              tpp[k][u] = gh[0];
              tux[k][u] = gh[NFP];
            }
          }
        }
      }
      // ---- B2: g''_b = sum_i grad(l_i) q_{b+e_i} / b!   (div u, grad p)
      {
        R lg[ET][12];  // grad(lambda) of the group's elements, hoisted into registers
#pragma unroll
        for (int u = 0; u < ET; ++u)
#pragma unroll
          for (int w = 0; w < 12; ++w) lg[u][w] = ld<R>(gb + u * EB + (C::O_GEO + w) * RB);
        const ushort4* vg = reinterpret_cast<const ushort4*>(tab + L.vg);
        for (int b = q; b < NPM1; b += TG) {
          const ushort4 o = __ldg(vg + b);
          const int off[4] = {o.x, o.y, o.z, o.w};
          const R sc = __ldg(invfacNm1 + b);
#pragma unroll
          for (int u = 0; u < ET; ++u) {
            const char* eb = gb + u * EB + C::X_Q * RB;
            R div = R(0), gx = R(0), gy = R(0), gz = R(0);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const R lx = lg[u][3 * j], ly = lg[u][3 * j + 1], lz = lg[u][3 * j + 2];
              const R pj = ld<R>(eb + off[j]);
              gx = fma(lx, pj, gx);
              gy = fma(ly, pj, gy);
              gz = fma(lz, pj, gz);
              div = fma(lx, ld<R>(eb + off[j] + NP * RB), div);
              div = fma(ly, ld<R>(eb + off[j] + 2 * NP * RB), div);
              div = fma(lz, ld<R>(eb + off[j] + 3 * NP * RB), div);
            }
            char* g = gb + u * EB + (C::X_G + 1 + b) * RB;
            st<R>(g, div * sc);
            st<R>(g + (NPM1 + 1) * RB, gx * sc);
            st<R>(g + 2 * (NPM1 + 1) * RB, gy * sc);
            st<R>(g + 3 * (NPM1 + 1) * RB, gz * sc);
          }
        }
      }
      auto flux_phase = [&]() {
      // ---- B1b: fluxes, F' = |grad l_f| c! F  (boundary: p+ = -p, u+ = u, R11)
#pragma unroll
      for (int k = 0; k < K1; ++k) {
        const int t = q + TG * k;
        const bool act = (NI1 % TG == 0) || t < NI1;
        const int tc = act ? t : 0;
        const int f = tc / NFP, i = tc - f * NFP;
        const int own = town[k];
        const R cs = __ldg(cfac + i);
#pragma unroll
        for (int u = 0; u < ET; ++u) {
          const char* eb = gb + u * EB + C::X_Q * RB;
          const int nb = reinterpret_cast<const int*>(gb + u * EB + 28 * RB)[f];
          const R pm = ld<R>(eb + own), uxm = ld<R>(eb + own + NP * RB), uym = ld<R>(eb + own + 2 * NP * RB),
                  uzm = ld<R>(eb + own + 3 * NP * RB);
          const bool bnd = (nb == -1) || !(act && u < nE);
          const R pp = bnd ? -pm : tpp[k][u], uxp = bnd ? uxm : tux[k][u], uyp = bnd ? uym : tuy[k][u],
                  uzp = bnd ? uzm : tuz[k][u];
          const char* gs = gb + u * EB + (C::O_GEO + 12 + 4 * f) * RB;
          const R nx = ld<R>(gs), ny = ld<R>(gs + RB), nz = ld<R>(gs + 2 * RB), sc = ld<R>(gs + 3 * RB) * cs;
          const R jp = pp - pm;
          const R jun = (nb < -1 && !A.gmap) ? -tux[k][u] - (nx * uxm + ny * uym + nz * uzm)
                                  : nx * (uxp - uxm) + ny * (uyp - uym) + nz * (uzp - uzm);
          if (act) {
            st<R>(gb + u * EB + (C::Y_F + (2 * f) * NFP + i) * RB, R(0.5) * sc * (A.tau_p * jp - jun));
            st<R>(gb + u * EB + (C::Y_F + (2 * f + 1) * NFP + i) * RB, R(0.5) * sc * (A.tau_u * jun - jp));
          }
        }
      }
      };
#if !BBW_FLUX_LATE
      flux_phase();
#endif
#if BBW_LSRK_REG
      // ---- B0: own Q -> registers (LSRK)
#pragma unroll
      for (int u = 0; u < ET; ++u)
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int k = 0; k < KO; ++k) {
            const int a = c == 0 ? BBW_PA(k) : q + TG * k;
            qo[u][c][k] = (q + TG * k < NP) ? ld<R>(gb + u * EB + (C::X_Q + c * NP + a) * RB) : R(0);
          }
#endif
#if BBW_LSRK_TMEM
      if (A.mode == 0) {  // park the LSRK state in TMEM until E / J
        R t0[TMR], t1[TMR];
#pragma unroll
        for (int i = 0; i < TMR; ++i) {
          t0[i] = i < 4 * KO ? rs[0][i / KO][i % KO] : R(0);
          t1[i] = i < 4 * KO ? qo[0][i / KO][i % KO] : R(0);
        }
        tm_store_reals<R, TMR>(taddr, 0, t0);
        tm_store_reals<R, TMR>(taddr, TMW, t1);
      }
#endif
      sync();
      BBW_PT(1);
      // ---- C1: r''_c[a] = -sum_j g''_c[a - e_j]  (p -> smem R_p, u -> registers)
      {
        const ushort4* ve = reinterpret_cast<const ushort4*>(tab + L.ve);
#pragma unroll
        for (int k = 0; k < KO; ++k) {
          const int a = q + TG * k;
          if (a < NP) {
            const ushort4 o = __ldg(ve + a);
            const char* p0 = gb + o.x + C::X_G * RB;
            const char* p1 = gb + o.y + C::X_G * RB;
            const char* p2 = gb + o.z + C::X_G * RB;
            const char* p3 = gb + o.w + C::X_G * RB;
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
              for (int u = 0; u < ET; ++u) {
                const int S = c * (NPM1 + 1) * RB + u * EB;
                const R v = (ld<R>(p0 + S) + ld<R>(p1 + S)) + (ld<R>(p2 + S) + ld<R>(p3 + S));
                if (c == 0) st<R>(gb + u * EB + (C::O_RP + a) * RB, -v);
                else ru[u][c - 1][k] = -v;
              }
          } else {
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
              for (int u = 0; u < ET; ++u) ru[u][c][k] = R(0);
          }
        }
      }
#if BBW_FLUX_LATE
      // the fluxes after the volume elevation: the neighbour-trace loads of B1a have B2 and C1 to arrive
      flux_phase();
      sync();
#endif
      // ---- C2: Y''[ff][d] = (sum_s F'[ff][d + e_s]) / (d!)^2
      face_sum3<C, R, NFP1, C::Y_F, NFP, C::Y_Y + 1, NFP1 + 1, true>(
          gb, q, reinterpret_cast<const ushort4*>(tab + L.trired) + trired_off(N - 1),
          reinterpret_cast<const R*>(tab + L.s_invf2));
      sync();
      BBW_PT(2);
      // ---- C3: layer 0: w'_0[c] = (2N+3) F'[c] + (c!)^2 sum_s Y''[c - e_s]
      {
        const ushort4* te = reinterpret_cast<const ushort4*>(tab + L.triele);
        const R* cf2 = reinterpret_cast<const R*>(tab + L.s_cf2);
        for (int c = q; c < NFP; c += TG) {
          const ushort4 o = __ldg(te + c);
          const R sc = __ldg(cf2 + c);
#pragma unroll
          for (int ff = 0; ff < 8; ++ff)
#pragma unroll
            for (int u = 0; u < ET; ++u) {
              const char* ya = gb + (C::Y_Y + ff * (NFP1 + 1)) * RB + u * EB;
              const R y = ld<R>(ya + o.x) + ld<R>(ya + o.y) + ld<R>(ya + o.z);
              const R F = ld<R>(gb + u * EB + (C::Y_F + ff * NFP + c) * RB);
              st<R>(gb + u * EB + (C::X_L + ff * C::FS + c) * RB, fma(sc, y, R(2 * N + 3) * F));
            }
        }
      }
      sync();
      BBW_PT(3);
      // LSRK inputs of u (Q_in and the residual, L2 hits) are issued now and consumed in E
#if BBW_LSRK_REG
#define BBW_QU(u, d, k) qo[u][1 + d][k]
#define BBW_SU(u, d, k) rs[u][1 + d][k]
#else
      R qu[ET][3][KO], su[ET][3][KO];
      if (A.mode == 0) {
#pragma unroll
        for (int u = 0; u < ET; ++u)
#pragma unroll
          for (int d = 0; d < 3; ++d)
#pragma unroll
            for (int k = 0; k < KO; ++k) {
              const int a = q + TG * k;
              const long long gi = (k0 + u) * 4 * NP + (1 + d) * NP + a;
              const bool ok = u < nE && a < NP;
              qu[u][d][k] = ok ? __ldg(A.Qin + gi) : R(0);
              su[u][d][k] = ok ? __ldcs(A.res + gi) : R(0);
            }
      }
#define BBW_QU(u, d, k) qu[u][d][k]
#define BBW_SU(u, d, k) su[u][d][k]
#endif
      // ---- D: lift layers j = 1..N: w'_j[d] = sum_s w'_{j-1}[d + e_s]
      if constexpr (C::ROWD) {
        // Row ownership: lane (ff, p) owns rows p and N - p (fixed c2, contiguous in c1) of face array ff at
        // every layer and keeps them in registers, so an output row needs only ONE other row from shared
        // memory (row c2 + 1 of the previous layer: the d + e2 operand; d + e0 and d + e1 are its own row)
        // instead of three operands per output.  Same arithmetic and summation order as face_sum3 (bitwise).
        constexpr int P = (N + 2) / 2;  // lanes per face array
        const int ff = q / P, p = q - ff * P;
        const bool act = ff < 8;
        const bool hasB = act && (N - p > p);
        const int rB = N - p;
        char* fa = gb + (C::X_L + (act ? ff : 0) * C::FS) * RB;
        R xa[N + 2], xb[P + 1];
        {
          const char* pa0 = fa + (p * (2 * N + 3 - p) / 2) * RB;
          const char* pb0 = fa + (rB * (2 * N + 3 - rB) / 2) * RB;
          static_for<0, N + 1, 1>([&](auto cc) {
            constexpr int c1 = decltype(cc)::value;
            if (act && c1 <= N - p) xa[c1] = ld<R>(pa0 + c1 * RB);
          });
          static_for<0, P, 1>([&](auto cc) {
            constexpr int c1 = decltype(cc)::value;
            if (hasB && c1 <= p) xb[c1] = ld<R>(pb0 + c1 * RB);
          });
        }
        static_for<1, N + 1, 1>([&](auto jc) {
          constexpr int j = decltype(jc)::value;
          constexpr int m = N - j;
          constexpr double MU = double(-j) / double(j + 1);
          if constexpr (j == 1) zero_region<C>(gb, q, C::Y_RPP, C::NS);  // padded r'' rows (F', Y'' are dead)
          // slot A: row p of degree m (p <= m), length m + 1 - p; operand row p + 1 of degree m + 1
          if (act && p <= m) {
            const char* ps = fa + (layer_off(N, j - 1) + (p + 1) * (2 * (m + 1) + 3 - (p + 1)) / 2) * RB;
            char* pd = fa + (layer_off(N, j) + p * (2 * m + 3 - p) / 2) * RB;
            R nb[m + 1];
            static_for<0, m + 1, 1>([&](auto cc) {
              constexpr int c1 = decltype(cc)::value;
              if (c1 <= m - p) nb[c1] = ld<R>(ps + c1 * RB);
            });
            static_for<0, m + 1, 1>([&](auto cc) {
              constexpr int c1 = decltype(cc)::value;
              if (c1 <= m - p) {
                R v = (xa[c1] + xa[c1 + 1]) + nb[c1];
                v *= R(MU);
                st<R>(pd + c1 * RB, v);
                xa[c1] = v;
              }
            });
          }
          // slot B: row N - p of degree m (needs p >= j), length p + 1 - j <= P - j; operand row N - p + 1
          if constexpr (P - j > 0) {
            if (hasB && p >= j) {
              const char* ps = fa + (layer_off(N, j - 1) + (rB + 1) * (2 * (m + 1) + 3 - (rB + 1)) / 2) * RB;
              char* pd = fa + (layer_off(N, j) + rB * (2 * m + 3 - rB) / 2) * RB;
              R nb[P - j];
              static_for<0, P - j, 1>([&](auto cc) {
                constexpr int c1 = decltype(cc)::value;
                if (c1 <= p - j) nb[c1] = ld<R>(ps + c1 * RB);
              });
              static_for<0, P - j, 1>([&](auto cc) {
                constexpr int c1 = decltype(cc)::value;
                if (c1 <= p - j) {
                  R v = (xb[c1] + xb[c1 + 1]) + nb[c1];
                  v *= R(MU);
                  st<R>(pd + c1 * RB, v);
                  xb[c1] = v;
                }
              });
            }
          }
          sync();
          BBW_PT(4);
        });
      } else
      static_for<1, N + 1, 1>([&](auto jc) {
        constexpr int j = decltype(jc)::value;
        constexpr int m = N - j;
        if constexpr (j == 1) zero_region<C>(gb, q, C::Y_RPP, C::NS);  // padded r'' rows (F', Y'' are dead)
        // layers are stored pre-multiplied by lam_j = (-1)^j/(j+1): s_j = -j/(j+1) R(s_{j-1}), s_0 = w'_0
        face_sum3<C, R, cnp2(m), C::X_L + layer_off(N, j - 1), NP, C::X_L + layer_off(N, j), NP, false, -j, j + 1>(
            gb, q, reinterpret_cast<const ushort4*>(tab + L.trired) + trired_off(m), static_cast<const R*>(nullptr));
        sync();
        BBW_PT(4);
      });
#if BBW_LSRK_TMEM
      if (A.mode == 0) {
        R t0[TMR], t1[TMR];
        tm_load_reals<R, TMR>(taddr, 0, t0);
        tm_load_reals<R, TMR>(taddr, TMW, t1);
#pragma unroll
        for (int i = 0; i < 4 * KO; ++i) {
          rs[0][i / KO][i % KO] = t0[i];
          qo[0][i / KO][i % KO] = t1[i];
        }
      }
#endif
      // ---- E: gather lifts; r''_p += S_p/(a!)^2 (+ source) -> smem; r_u = a! r''_u + S_u/a!; LSRK for u
      //      r''_p also goes to a zero-padded row copy (row stride N+1) in the dead face region for F
      {
        const uint16_t* padoff = reinterpret_cast<const uint16_t*>(tab + L.padoff);
        R nrm[ET][12];  // outward normals of the group's elements, hoisted into registers
#pragma unroll
        for (int u = 0; u < ET; ++u)
#pragma unroll
          for (int f = 0; f < 4; ++f)
#pragma unroll
            for (int dd = 0; dd < 3; ++dd) nrm[u][3 * f + dd] = ld<R>(gb + u * EB + (C::O_GEO + 12 + 4 * f + dd) * RB);
        const uint2* lgt = reinterpret_cast<const uint2*>(tab + L.lg);
#pragma unroll
        for (int k = 0; k < KO; ++k) {
          const int a = q + TG * k;
          if (a < NP) {
            const uint2 e = __ldg(lgt + a);
            const int lo[4] = {(int)(e.x & 0xFFFF), (int)(e.x >> 16), (int)(e.y & 0xFFFF), (int)(e.y >> 16)};

            const R i1 = __ldg(invfacN + a), i2 = i1 * i1, f1 = __ldg(facN + a);  // 1/a!, 1/(a!)^2, a!
            const int pado = __ldg(padoff + a);
#pragma unroll
            for (int u = 0; u < ET; ++u) {
              const char* eb = gb + u * EB;
              R sp = R(0), sx = R(0), sy = R(0), sz = R(0);
#pragma unroll
              for (int f = 0; f < 4; ++f) {
                const R wp = ld<R>(eb + (C::X_L + (2 * f) * C::FS) * RB + lo[f]);  // lam_{a_f} already applied (D)
                const R wu = ld<R>(eb + (C::X_L + (2 * f + 1) * C::FS) * RB + lo[f]);
                sp += wp;
                sx = fma(nrm[u][3 * f], wu, sx);
                sy = fma(nrm[u][3 * f + 1], wu, sy);
                sz = fma(nrm[u][3 * f + 2], wu, sz);
              }
              const long long kk = k0 + u;
              R rp = fma(sp, i2, ld<R>(eb + (C::O_RP + a) * RB));
              if (A.src && u < nE) rp = fma(A.src_amp * __ldg(A.src + kk * NP + a), i1, rp);
              st<R>(gb + u * EB + (C::O_RP + a) * RB, rp);
              st<R>(gb + u * EB + C::Y_RPP * RB + pado, rp);
              const R r3[3] = {fma(ru[u][0][k], f1, sx * i1), fma(ru[u][1][k], f1, sy * i1),
                               fma(ru[u][2][k], f1, sz * i1)};
              if (u < nE) {
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                  const long long gi = kk * 4 * NP + (1 + d) * NP + a;
                  if (A.mode == 0) {
                    const R r = fma(A.rk_a, BBW_SU(u, d, k), A.dt * r3[d]);
                    st_out(A.res + gi, r);
                    st_out(A.Qout + gi, fma(A.rk_b, r, BBW_QU(u, d, k)));
                  } else {
                    A.Qout[gi] = r3[d];
                  }
                }
              }
            }
          }
        }
      }
      sync();
      BBW_PT(5);
    }

    // ---- F-I: WADG multiply + telescoping projection of r_p
    R osc[KO];  // TRIPLE: b_N at the lane's shell slots; v4: the output scales a!/N!
    constexpr bool M0FAST = (M == 0) && BBW_M0_FAST;
    if constexpr (M0FAST) {
      // M = 0 (piecewise-constant c^2, BBDG): P^N_N = I (c_0 = 1, c_j = 0 for j >= 1), so the WADG
      // update is the multiplication of r_p by the element's constant c^2: dp/dt_a = c^2 a! r''_p[a]; the
      // product and the telescoping sweeps are skipped
      const R c0 = ld<R>(gb + C::O_C * RB);
#pragma unroll
      for (int k = 0; k < KO; ++k) osc[k] = c0 * __ldg(facN + cmin(q + TG * k, NP - 1));
    } else {
      wadg_phases<C, R>(gb, q, A, sync, pt_prev, osc);
    }
    constexpr int RES = M0FAST ? C::O_RP : C::TRIPLE ? C::tlev(N) : wadg_result<C>();
    // TRIPLE: shell index (layout.hpp) of the lane's canonical coefficients a = q + TG k, where J reads b_N
    int cshk[KO];
#pragma unroll
    for (int k = 0; k < KO; ++k)
      cshk[k] = (C::TRIPLE && !M0FAST)
                    ? (int)__ldg(reinterpret_cast<const uint32_t*>(tab + L.sho) + cmin(q + TG * k, NP - 1))
                    : q + TG * k;

    // ---- J: dp/dt = a!/N! b_N; outputs
#if BBW_LSRK_TMEM
    if (A.mode == 0) {
      R t0[TMR], t1[TMR];
      tm_load_reals<R, TMR>(taddr, 0, t0);
      tm_load_reals<R, TMR>(taddr, TMW, t1);
#pragma unroll
      for (int i = 0; i < KO; ++i) {
        rs[0][0][i] = t0[i];
        qo[0][0][i] = t1[i];
      }
    }
#endif
#if BBW_LSRK_REG
#define BBW_QP(u, k) qo[u][0][k]
#define BBW_SP(u, k) rs[u][0][k]
#else
    R qp[ET][KO], sp[ET][KO];
    if (A.mode == 0) {
#pragma unroll
      for (int u = 0; u < ET; ++u)
#pragma unroll
        for (int k = 0; k < KO; ++k) {
          const int a = BBW_PA(k);
          const long long gi = (k0 + u) * 4 * NP + a;
          const bool ok = u < nE && q + TG * k < NP;
          qp[u][k] = ok ? __ldg(A.Qin + gi) : R(0);
          sp[u][k] = ok ? __ldcs(A.res + gi) : R(0);
        }
    }
#define BBW_QP(u, k) qp[u][k]
#define BBW_SP(u, k) sp[u][k]
#endif
#pragma unroll
    for (int k = 0; k < KO; ++k) {
      const int a = BBW_PA(k);
      if (q + TG * k < NP) {
        const R sc = (C::TRIPLE && !M0FAST) ? __ldg(outN + a) : osc[k];  // a!/N! (M0FAST: c^2 a!)
#pragma unroll
        for (int u = 0; u < ET; ++u) {
          if (u >= nE) continue;
          const long long kk = k0 + u;
          const R dp = ld<R>(gb + u * EB + (RES + cshk[k]) * RB) * sc;
          if (A.mode == 2) {
            A.Qout[kk * NP + a] = dp;
          } else {
            const long long gi = kk * 4 * NP + a;
            if (A.mode == 0) {
              const R r = fma(A.rk_a, BBW_SP(u, k), A.dt * dp);
              st_out(A.res + gi, r);
              st_out(A.Qout + gi, fma(A.rk_b, r, BBW_QP(u, k)));
            } else {
              A.Qout[gi] = dp;
            }
          }
        }
      }
    }
    if constexpr (kTMA) fence_proxy_async();  // this batch's generic smem accesses before the next batch's bulk writes
    sync();
    BBW_PT(10);
  }
#if BBW_DYNQ
  {
    // every unit has drawn its failing ticket before it counts itself done: the last one resets the queue
    const bool leader = (TG <= 32) ? ((tid & 31) == 0) : (q == 0);
    if (leader) {
      const unsigned units = gridDim.x * (TG <= 32 ? C::T / 32 : C::G);
      __threadfence();
      if (atomicAdd(A.qctr + 1, 1u) == units - 1) {
        A.qctr[0] = 0;
        A.qctr[1] = 0;
        __threadfence();
      }
    }
  }
#endif
#if BBW_LSRK_TMEM
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_s), "r"(TMCOLS) : "memory");
#endif
}

// Halo pack: for each send face (local element k, face f) write the two traces the
// receiver's flux needs (Eq. sdf), in the sender's canonical face ordering:
//   buf[slot][0][i] = p(face node i),   buf[slot][1][i] = u(face node i) . n_f,
// n_f = -grad(lambda_f)/|grad(lambda_f)| the sender's outward unit normal (2 Nfp words per face).
template <int N, typename R>
__global__ void pack_kernel(const R* __restrict__ Q, const R* __restrict__ geo, const int* __restrict__ faces,
                            int nfaces, const uint16_t* __restrict__ fnode_bytes, R* __restrict__ buf) {
  constexpr int NP = cnp3(N), NFP = cnp2(N);
  const long long total = (long long)nfaces * NFP;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int slot = (int)(t / NFP), i = (int)(t - (long long)slot * NFP);
    const int k = faces[2 * slot], f = faces[2 * slot + 1];
    const R* g = geo + (long long)k * 12 + 3 * f;
    const R gx = g[0], gy = g[1], gz = g[2];
    const R il = R(1) / sqrt(gx * gx + gy * gy + gz * gz);
    const R* qk = Q + (long long)k * 4 * NP + __ldg(fnode_bytes + f * NFP + i) / (int)sizeof(R);
    R* b = buf + (long long)slot * 2 * NFP + i;
    b[0] = qk[0];
    b[NFP] = (-gx * il) * qk[NP] + (-gy * il) * qk[2 * NP] + (-gz * il) * qk[3 * NP];
  }
}

}  // namespace bbw
