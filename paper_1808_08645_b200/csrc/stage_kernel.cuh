// Fused BBWADG RK-stage kernel for sm_100a, v2 (templated on N, M and the real type).
//
// One persistent CTA processes batches of E = G x ET consecutive elements (Morton order, so
// neighbour traces are mostly L2-resident).  The CTA's threads form G groups; a thread of group
// g computes output coefficient i of a phase for the ET elements g*ET .. g*ET+ET-1 at once, so
// each table lookup (neighbour byte offsets) is shared by ET elements and every shared-memory
// address is "table register + compile-time immediate" (array base + element stride).
//
// All one-degree Bernstein reductions/elevations run as UNWEIGHTED 4-point sums in factorial-
// scaled variables (layout.hpp), with the 1/n and c_j factors folded into per-level constants:
//   A  load Q_in (16-B vectors), c^2_M / beta!, grad(lambda) and face normals
//   B  surface fluxes F_p, F_u scaled by |grad lambda_f| c!;
//      degree-(N-1) gradient g''_b = sum_i grad(lambda_i) q_{b+e_i} / b!
//   C  volume r''_a = -sum_j g''_{a-e_j} (elevation, x/a! scaling); L_0 F as
//      reduction -> 1/(d!)^2 -> elevation -> (c!)^2
//   D  N face reductions -> lift layers w_j
//   E  gather the 4 lifts into r; LSRK update of u_x, u_y, u_z (streamed to HBM)
//   F  Bernstein product h'_g = (g!)^2 N!M!/(N+M)! sum r''_a c''_b  (Eq. mcoeff)
//   G  M reductions N+M -> N;  H  N downward reductions;  I  N upward elevations with the
//      level constants gam_n = (n!)^2 c_{N-n}/(N+M)!  (telescoping form, Eq. telescope)
//   J  dp/dt_a = a!/N! b_N[a];  LSRK update of p
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
__host__ __device__ constexpr int pow2_floor(int x) { return x >= 32 ? 32 : x >= 16 ? 16 : x >= 8 ? 8 : x >= 4 ? 4 : x >= 2 ? 2 : 1; }

template <typename R>
struct StageArgs {
  const R* Qin;
  R* Qout;
  R* res;
  const R* c2;
  const R* geo;        // [K][12]: grad(lambda_0..3)
  const int* nbr;      // [K][4]
  const uint8_t* code; // [K][4] = 6 f' + sigma
  const R* ghost;      // [slots][4][NFP]
  const R* src;        // [K][NP] or null
  const uint8_t* tab;  // table blob (layout.hpp)
  long long elem_begin, elem_end;
  R rk_a, rk_b, dt, src_amp, tau_p, tau_u;
  R gam[10], lam[10];
  int mode;  // 0 LSRK stage, 1 write dQ/dt into Qout, 2 WADG apply (Qin=r[K][NP] -> Qout[K][NP])
};

template <int N_, int M_, typename R>
struct StageCfg {
  static constexpr int N = N_, M = M_;
  static constexpr int NP = cnp3(N), NFP = cnp2(N), NFP1 = cnp2(N - 1), MP = cnp3(M), NPH = cnp3(N + M);
  static constexpr int NPM1 = cnp3(N - 1), NP4 = cnp4(N);
  static constexpr int RB = (int)sizeof(R);
#ifndef BBW_T
#define BBW_T 256
#endif
#ifndef BBW_SMEM_KB
#define BBW_SMEM_KB 110
#endif
  static constexpr int T = BBW_T;
  static constexpr int VEC = 16 / RB;
  // ---- per-element shared-memory layout (in reals)
  static constexpr int O_Q = 0, O_R = 4 * NP, O_RS = 8 * NP, O_GEO = 12 * NP, O_C = O_GEO + 32;
  static constexpr int O_W = rup(O_C + MP, 2);
  // surface phase
  static constexpr int S_G = O_W;                      // 4 x [zero, NPM1]
  static constexpr int S_F = S_G + 4 * (NPM1 + 1);     // 8 x [NFP]  (face f, flux p/u)
  static constexpr int S_Y = S_F + 8 * NFP;            // 8 x [zero, NFP1]
  static constexpr int S_L = S_Y + 8 * (NFP1 + 1);     // 8 x [NP]   lift layers
  static constexpr int S_END = S_L + 8 * NP;
  // WADG phase
  static constexpr int W_H = O_W, W_P = W_H + NPH, W_LEV = W_P + NPH;
  static constexpr int W_A0 = W_LEV + NP4, W_A1 = W_A0 + NP + 1;
  static constexpr int W_END = W_A1 + NP + 1;
  static constexpr int PER_E = rup(cmax(S_END, W_END), VEC);
  static constexpr int EB = PER_E * RB;  // element stride in bytes
  // ---- batching
#ifdef BBW_ET
  static constexpr int ET = BBW_ET;
#else
  static constexpr int ET = (N <= 3) ? 4 : 2;  // elements per thread (share one table lookup)
#endif
  static constexpr int SMEM_TARGET = BBW_SMEM_KB * 1024;
  static constexpr int G = cmin(T / 8, pow2_floor(cmax(1, SMEM_TARGET / (ET * EB))));
  static constexpr int E = G * ET;
  static constexpr int TG = T / G;
  static constexpr int SMEM_BYTES = E * EB;
  static_assert(TG >= 8, "too many groups");
};

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

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

// one pure 4-point (or 3-point) sum stencil phase over CNT outputs:
//   dst[i] = SCALE(i) * sum_j src[off_j(i)]   for the ET elements of the thread's group
template <class C, typename R, int CNT, int SRC, int DST, int NTERMS>
__device__ __forceinline__ void sum_phase(char* gb, int q, const ushort4* __restrict__ tab) {
#pragma unroll 2
  for (int i = q; i < CNT; i += C::TG) {
    const ushort4 o = __ldg(tab + i);
    const char* p0 = gb + o.x;
    const char* p1 = gb + o.y;
    const char* p2 = gb + o.z;
    const char* p3 = gb + o.w;
#pragma unroll
    for (int u = 0; u < C::ET; ++u) {
      constexpr int S = SRC * C::RB;
      R v = ld<R>(p0 + S + u * C::EB) + ld<R>(p1 + S + u * C::EB) + ld<R>(p2 + S + u * C::EB);
      if constexpr (NTERMS == 4) v += ld<R>(p3 + S + u * C::EB);
      st<R>(gb + DST * C::RB + u * C::EB + i * C::RB, v);
    }
  }
}

template <class C, typename R>
__device__ __forceinline__ void wadg_phases(char* gb, int q, const StageArgs<R>& A) {
  constexpr int N = C::N, M = C::M, NP = C::NP, NPH = C::NPH, RB = C::RB, ET = C::ET, EB = C::EB, TG = C::TG;
  const TabLayout L = tab_layout(N, M, RB);
  const uint8_t* tab = A.tab;
  const int* csr_ptr = reinterpret_cast<const int*>(tab + L.csr_ptr);
  const uint32_t* csr = reinterpret_cast<const uint32_t*>(tab + L.csr_terms);
  const R* post = reinterpret_cast<const R*>(tab + L.s_post);
  const ushort4* red = reinterpret_cast<const ushort4*>(tab + L.red);

  // F: h'_g = post_g * sum_{a+b=g} r''_a c''_b
  for (int g = q; g < NPH; g += TG) {
    const int t0 = __ldg(csr_ptr + g), t1 = __ldg(csr_ptr + g + 1);
    R acc[ET];
#pragma unroll
    for (int u = 0; u < ET; ++u) acc[u] = R(0);
#pragma unroll 4
    for (int t = t0; t < t1; ++t) {
      const uint32_t w = __ldg(csr + t);
      const char* pa = gb + (w & 0xFFFF) + C::O_R * RB;
      const char* pb = gb + (w >> 16) + C::O_C * RB;
#pragma unroll
      for (int u = 0; u < ET; ++u) acc[u] = fma(ld<R>(pa + u * EB), ld<R>(pb + u * EB), acc[u]);
    }
    const R s = __ldg(post + g);
#pragma unroll
    for (int u = 0; u < ET; ++u) st<R>(gb + (C::W_H + g) * RB + u * EB, acc[u] * s);
  }
  if (q == 0) {
#pragma unroll
    for (int u = 0; u < ET; ++u) {
      st<R>(gb + C::W_A0 * RB + u * EB, R(0));
      st<R>(gb + C::W_A1 * RB + u * EB, R(0));
    }
  }
  __syncthreads();

  // G: M reductions N+M -> N (ping-pong H <-> P; the last lands in level N)
  static_for<N + M, N, -1>([&](auto nc) {
    constexpr int n = decltype(nc)::value;
    constexpr int k = N + M - n;  // iteration index
    constexpr int SRC = (k % 2 == 0) ? C::W_H : C::W_P;
    constexpr int DST = (n - 1 == N) ? C::W_LEV + cnp4(N - 1) : ((k % 2 == 0) ? C::W_P : C::W_H);
    sum_phase<C, R, cnp3(n - 1), SRC, DST, 4>(gb, q, red + red_off(n));
    __syncthreads();
  });
  if constexpr (M == 0) {
    for (int i = q; i < NP; i += TG)
#pragma unroll
      for (int u = 0; u < ET; ++u)
        st<R>(gb + (C::W_LEV + cnp4(N - 1) + i) * RB + u * EB, ld<R>(gb + (C::W_H + i) * RB + u * EB));
    __syncthreads();
  }
  // H: downward reductions level n -> n-1 (pure sums); seed b_0 = gam_0 u_0 in A0[1]
  static_for<N, 0, -1>([&](auto nc) {
    constexpr int n = decltype(nc)::value;
    sum_phase<C, R, cnp3(n - 1), C::W_LEV + cnp4(n - 1), C::W_LEV + cnp4(n - 2), 4>(gb, q, red + red_off(n));
    __syncthreads();
  });
  if (q == 0) {
#pragma unroll
    for (int u = 0; u < ET; ++u) st<R>(gb + (C::W_A0 + 1) * RB + u * EB, A.gam[0] * ld<R>(gb + C::W_LEV * RB + u * EB));
  }
  __syncthreads();
  // I: upward: b_n[a] = sum_j b_{n-1}[a - e_j] + gam_n / (a!)^2 u_n[a]   (b_n in A_{n%2})
  static_for<1, N + 1, 1>([&](auto nc) {
    constexpr int n = decltype(nc)::value;
    constexpr int SRC = (n % 2 == 1) ? C::W_A0 : C::W_A1;
    constexpr int DST = (n % 2 == 1) ? C::W_A1 : C::W_A0;
    const R gn = A.gam[n];
    const uint8_t* up = tab + L.upw + 16 * upw_off(n);
    for (int i = q; i < cnp3(n); i += TG) {
      const ushort4 o = __ldg(reinterpret_cast<const ushort4*>(up + 16 * i));
      const R w = gn * __ldg(reinterpret_cast<const R*>(up + 16 * i + 8));
      const char* p0 = gb + o.x;
      const char* p1 = gb + o.y;
      const char* p2 = gb + o.z;
      const char* p3 = gb + o.w;
#pragma unroll
      for (int u = 0; u < ET; ++u) {
        constexpr int S = SRC * RB;
        R v = (ld<R>(p0 + S + u * EB) + ld<R>(p1 + S + u * EB)) + (ld<R>(p2 + S + u * EB) + ld<R>(p3 + S + u * EB));
        v = fma(w, ld<R>(gb + (C::W_LEV + cnp4(n - 1) + i) * RB + u * EB), v);
        st<R>(gb + (DST + 1 + i) * RB + u * EB, v);
      }
    }
    __syncthreads();
  });
}

template <class C>
__host__ __device__ constexpr int wadg_result() {
  return (C::N % 2 == 1) ? C::W_A1 + 1 : C::W_A0 + 1;
}

template <class C, typename R>
__global__ void __launch_bounds__(C::T) stage_kernel(const StageArgs<R> A) {
  constexpr int N = C::N, M = C::M, NP = C::NP, NFP = C::NFP, NFP1 = C::NFP1, MP = C::MP, NPM1 = C::NPM1;
  constexpr int E = C::E, T = C::T, ET = C::ET, EB = C::EB, RB = C::RB, TG = C::TG, VEC = C::VEC;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ R lam_s[10];
  char* smem = reinterpret_cast<char*>(smem_raw);
  const int tid = threadIdx.x;
  if (tid < 10) lam_s[tid] = A.lam[tid < 9 ? tid : 9];
  const int grp = tid / TG, q = tid - grp * TG;
  char* gb = smem + grp * ET * EB;  // this thread's group base
  const TabLayout L = tab_layout(N, M, RB);
  const uint8_t* tab = A.tab;
  const R* invfacN = reinterpret_cast<const R*>(tab + L.s_invfacN);
  const R* facN = reinterpret_cast<const R*>(tab + L.s_facN);
  const R* invfac2N = reinterpret_cast<const R*>(tab + L.s_invfac2N);
  const R* outN = reinterpret_cast<const R*>(tab + L.s_outN);
  const R* invfacM = reinterpret_cast<const R*>(tab + L.s_invfacM);
  const R* invfacNm1 = reinterpret_cast<const R*>(tab + L.s_invfacNm1);
  const R* cfac = reinterpret_cast<const R*>(tab + L.s_cfac);
  const R* invf2 = reinterpret_cast<const R*>(tab + L.s_invf2);
  const R* cf2 = reinterpret_cast<const R*>(tab + L.s_cf2);
  const uint16_t* fnode = reinterpret_cast<const uint16_t*>(tab + L.fnode);
  const uint16_t* nbrvol = reinterpret_cast<const uint16_t*>(tab + L.nbrvol);
  const uint16_t* nbrface = reinterpret_cast<const uint16_t*>(tab + L.nbrface);

  const long long nelem = A.elem_end - A.elem_begin;
  const long long nbatch = (nelem + E - 1) / E;
  for (long long batch = blockIdx.x; batch < nbatch; batch += gridDim.x) {
    const long long e0 = A.elem_begin + batch * E;
    const int nE = (int)((A.elem_end - e0) < E ? (A.elem_end - e0) : E);
    const long long k0 = e0 + grp * ET;  // first element of this thread's group

    // ---- A: loads.  The LSRK residual of the batch is prefetched asynchronously (cp.async,
    //      waited for before phase E) so its HBM latency overlaps the surface/volume phases.
    if (A.mode == 0) {
      constexpr int NV = 4 * NP / VEC;
      const char* gr = reinterpret_cast<const char*>(A.res + e0 * 4 * NP);
      for (int t = tid; t < nE * NV; t += T) {
        const int e = t / NV, w = t - e * NV;
        cp_async16(smem + e * EB + C::O_RS * RB + w * 16, gr + (size_t)t * 16);
      }
      cp_async_commit();
    }
    if (A.mode == 2) {
      for (int t = tid; t < nE * NP; t += T) {
        const int e = t / NP, a = t - e * NP;
        st<R>(smem + e * EB + (C::O_R + a) * RB, A.Qin[(e0 + e) * NP + a] * __ldg(invfacN + a));
      }
    } else {
      constexpr int NV = 4 * NP / VEC;
      using V = typename std::conditional<sizeof(R) == 8, double2, float4>::type;
      const V* gq = reinterpret_cast<const V*>(A.Qin + e0 * 4 * NP);
      for (int t = tid; t < nE * NV; t += T) {
        const int e = t / NV, w = t - e * NV;
        *reinterpret_cast<V*>(smem + e * EB + w * 16) = gq[t];
      }
      for (int t = tid; t < nE * 4; t += T) {  // grad lambda_f, |grad lambda_f|, outward normal
        const int e = t >> 2, f = t & 3;
        const R* gg = A.geo + (e0 + e) * 12 + 3 * f;
        const R gx = gg[0], gy = gg[1], gz = gg[2];
        const R gl = sqrt(gx * gx + gy * gy + gz * gz), il = R(1) / gl;
        char* s = smem + e * EB + C::O_GEO * RB;
        st<R>(s + (3 * f) * RB, gx);
        st<R>(s + (3 * f + 1) * RB, gy);
        st<R>(s + (3 * f + 2) * RB, gz);
        st<R>(s + (12 + 4 * f) * RB, -gx * il);
        st<R>(s + (13 + 4 * f) * RB, -gy * il);
        st<R>(s + (14 + 4 * f) * RB, -gz * il);
        st<R>(s + (15 + 4 * f) * RB, gl);
      }
      for (int t = tid; t < E * 12; t += T) {  // zero slots of G'' (4) and Y'' (8) arrays
        const int e = t / 12, z = t - e * 12;
        const int off = z < 4 ? C::S_G + z * (NPM1 + 1) : C::S_Y + (z - 4) * (NFP1 + 1);
        st<R>(smem + e * EB + off * RB, R(0));
      }
    }
    for (int t = tid; t < nE * MP; t += T) {
      const int e = t / MP, b = t - e * MP;
      st<R>(smem + e * EB + (C::O_C + b) * RB, A.c2[(e0 + e) * MP + b] * __ldg(invfacM + b));
    }
    __syncthreads();

    if (A.mode != 2) {
      // ---- B1: fluxes, F' = |grad l_f| c! F
      for (int t = q; t < 4 * NFP; t += TG) {
        const int f = t / NFP, i = t - f * NFP;
        const int own = __ldg(fnode + f * NFP + i);
        const R cs = __ldg(cfac + i);
#pragma unroll
        for (int u = 0; u < ET; ++u) {
          const char* eb = gb + u * EB;
          const long long k = k0 + u;
          R pm = ld<R>(eb + own), uxm = ld<R>(eb + own + NP * RB), uym = ld<R>(eb + own + 2 * NP * RB),
            uzm = ld<R>(eb + own + 3 * NP * RB);
          R pp = -pm, uxp = uxm, uyp = uym, uzp = uzm;
          if (k < A.elem_end) {
            const int nb = __ldg(A.nbr + k * 4 + f);
            if (nb >= 0) {
              const int vol = __ldg(nbrvol + __ldg(A.code + k * 4 + f) * NFP + i);
              const R* qn = A.Qin + (long long)nb * 4 * NP + vol;
              pp = __ldg(qn);
              uxp = __ldg(qn + NP);
              uyp = __ldg(qn + 2 * NP);
              uzp = __ldg(qn + 3 * NP);
            } else if (nb < -1) {
              const int fi = __ldg(nbrface + (__ldg(A.code + k * 4 + f) % 6) * NFP + i);
              const R* gh = A.ghost + (long long)(-2 - nb) * 4 * NFP + fi;
              pp = gh[0];
              uxp = gh[NFP];
              uyp = gh[2 * NFP];
              uzp = gh[3 * NFP];
            }
          }
          const char* gs = eb + (C::O_GEO + 12 + 4 * f) * RB;
          const R nx = ld<R>(gs), ny = ld<R>(gs + RB), nz = ld<R>(gs + 2 * RB), sc = ld<R>(gs + 3 * RB) * cs;
          const R jp = pp - pm;
          const R jun = nx * (uxp - uxm) + ny * (uyp - uym) + nz * (uzp - uzm);
          st<R>(gb + u * EB + (C::S_F + (2 * f) * NFP + i) * RB, R(0.5) * sc * (A.tau_p * jp - jun));
          st<R>(gb + u * EB + (C::S_F + (2 * f + 1) * NFP + i) * RB, R(0.5) * sc * (A.tau_u * jun - jp));
        }
      }
      // ---- B2: g''_b = sum_i grad(l_i) q_{b+e_i} / b!   (div u, grad p)
      {
        R lg[ET][12];
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
            const char* eb = gb + u * EB;
            R div = R(0), gx = R(0), gy = R(0), gz = R(0);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const R pj = ld<R>(eb + off[j]);
              gx = fma(lg[u][3 * j], pj, gx);
              gy = fma(lg[u][3 * j + 1], pj, gy);
              gz = fma(lg[u][3 * j + 2], pj, gz);
              div = fma(lg[u][3 * j], ld<R>(eb + off[j] + NP * RB), div);
              div = fma(lg[u][3 * j + 1], ld<R>(eb + off[j] + 2 * NP * RB), div);
              div = fma(lg[u][3 * j + 2], ld<R>(eb + off[j] + 3 * NP * RB), div);
            }
            char* g = gb + u * EB + (C::S_G + 1 + b) * RB;
            st<R>(g, div * sc);
            st<R>(g + (NPM1 + 1) * RB, gx * sc);
            st<R>(g + 2 * (NPM1 + 1) * RB, gy * sc);
            st<R>(g + 3 * (NPM1 + 1) * RB, gz * sc);
          }
        }
      }
      __syncthreads();
      // ---- C1: r''_c[a] = -sum_j g''_c[a - e_j]   (4 fields; zero slot for a_j = 0)
      {
        const ushort4* ve = reinterpret_cast<const ushort4*>(tab + L.ve);
        for (int a = q; a < NP; a += TG) {
          const ushort4 o = __ldg(ve + a);
          const char* p0 = gb + o.x;
          const char* p1 = gb + o.y;
          const char* p2 = gb + o.z;
          const char* p3 = gb + o.w;
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int u = 0; u < ET; ++u) {
              constexpr int S0 = C::S_G * RB;
              const int S = S0 + c * (NPM1 + 1) * RB + u * EB;
              const R v = (ld<R>(p0 + S) + ld<R>(p1 + S)) + (ld<R>(p2 + S) + ld<R>(p3 + S));
              st<R>(gb + u * EB + (C::O_R + c * NP + a) * RB, -v);
            }
        }
      }
      // ---- C2: y''[d] = (sum_s F'[d + e_s]) / (d!)^2   (8 face arrays)
      {
        const ushort4* tr = reinterpret_cast<const ushort4*>(tab + L.trired) + trired_off(N - 1);
        for (int t = q; t < 8 * NFP1; t += TG) {
          const int ff = t / NFP1, d = t - ff * NFP1;
          const ushort4 o = __ldg(tr + d);
          const R sc = __ldg(invf2 + d);
          const char* fa = gb + (C::S_F + ff * NFP) * RB;
#pragma unroll
          for (int u = 0; u < ET; ++u) {
            const R v = ld<R>(fa + o.x + u * EB) + ld<R>(fa + o.y + u * EB) + ld<R>(fa + o.z + u * EB);
            st<R>(gb + u * EB + (C::S_Y + ff * (NFP1 + 1) + 1 + d) * RB, v * sc);
          }
        }
      }
      __syncthreads();
      // ---- C3: layer 0: w'_0[c] = (2N+3) F'[c] + (c!)^2 sum_s y''[c - e_s]
      {
        const ushort4* te = reinterpret_cast<const ushort4*>(tab + L.triele);
        for (int t = q; t < 8 * NFP; t += TG) {
          const int ff = t / NFP, c = t - ff * NFP;
          const ushort4 o = __ldg(te + c);
          const R sc = __ldg(cf2 + c);
          const char* ya = gb + (C::S_Y + ff * (NFP1 + 1)) * RB;
#pragma unroll
          for (int u = 0; u < ET; ++u) {
            const R y = ld<R>(ya + o.x + u * EB) + ld<R>(ya + o.y + u * EB) + ld<R>(ya + o.z + u * EB);
            const R F = ld<R>(gb + u * EB + (C::S_F + ff * NFP + c) * RB);
            st<R>(gb + u * EB + (C::S_L + ff * NP + c) * RB, fma(sc, y, R(2 * N + 3) * F));
          }
        }
      }
      __syncthreads();
      // ---- D: lift layers j = 1..N: w'_j[d] = sum_s w'_{j-1}[d + e_s]
      static_for<1, N + 1, 1>([&](auto jc) {
        constexpr int j = decltype(jc)::value;
        constexpr int m = N - j, CNT = cnp2(m);
        const ushort4* tr = reinterpret_cast<const ushort4*>(tab + L.trired) + trired_off(m);
        for (int t = q; t < 8 * CNT; t += TG) {
          const int ff = t / CNT, d = t - ff * CNT;
          const ushort4 o = __ldg(tr + d);
          const char* la = gb + (C::S_L + ff * NP + layer_off(N, j - 1)) * RB;
#pragma unroll
          for (int u = 0; u < ET; ++u) {
            const R v = ld<R>(la + o.x + u * EB) + ld<R>(la + o.y + u * EB) + ld<R>(la + o.z + u * EB);
            st<R>(gb + u * EB + (C::S_L + ff * NP + layer_off(N, j) + d) * RB, v);
          }
        }
        __syncthreads();
      });
      // ---- E: gather lifts; r''_p += S_p/(a!)^2 (+ source); r_u = a! r''_u + S_u/a!; LSRK for u
      if (A.mode == 0) {
        cp_async_wait_all();
        __syncthreads();
      }
      {
        R nrm[ET][12];
#pragma unroll
        for (int u = 0; u < ET; ++u)
#pragma unroll
          for (int f = 0; f < 4; ++f)
#pragma unroll
            for (int d = 0; d < 3; ++d) nrm[u][3 * f + d] = ld<R>(gb + u * EB + (C::O_GEO + 12 + 4 * f + d) * RB);
        const uint4* lgt = reinterpret_cast<const uint4*>(tab + L.lg);
        for (int a = q; a < NP; a += TG) {
          const uint4 e = __ldg(lgt + a);
          const int lo[4] = {(int)(e.x & 0xFFFF), (int)(e.x >> 16), (int)(e.y & 0xFFFF), (int)(e.y >> 16)};
          R lm[4];
#pragma unroll
          for (int f = 0; f < 4; ++f) lm[f] = lam_s[(e.z >> (8 * f)) & 0xFF];
          const R i1 = __ldg(invfacN + a), i2 = __ldg(invfac2N + a), f1 = __ldg(facN + a);
#pragma unroll
          for (int u = 0; u < ET; ++u) {
            const char* eb = gb + u * EB;
            R sp = R(0), sx = R(0), sy = R(0), sz = R(0);
#pragma unroll
            for (int f = 0; f < 4; ++f) {
              const R wp = lm[f] * ld<R>(eb + (C::S_L + (2 * f) * NP) * RB + lo[f]);
              const R wu = lm[f] * ld<R>(eb + (C::S_L + (2 * f + 1) * NP) * RB + lo[f]);
              sp += wp;
              sx = fma(nrm[u][3 * f], wu, sx);
              sy = fma(nrm[u][3 * f + 1], wu, sy);
              sz = fma(nrm[u][3 * f + 2], wu, sz);
            }
            const long long k = k0 + u;
            R rp = fma(sp, i2, ld<R>(eb + (C::O_R + a) * RB));
            if (A.src && k < A.elem_end) rp = fma(A.src_amp * A.src[k * NP + a], i1, rp);
            st<R>(gb + u * EB + (C::O_R + a) * RB, rp);
            const R ru[3] = {fma(ld<R>(eb + (C::O_R + NP + a) * RB), f1, sx * i1),
                             fma(ld<R>(eb + (C::O_R + 2 * NP + a) * RB), f1, sy * i1),
                             fma(ld<R>(eb + (C::O_R + 3 * NP + a) * RB), f1, sz * i1)};
            if (k < A.elem_end) {
#pragma unroll
              for (int d = 0; d < 3; ++d) {
                const long long gi = k * 4 * NP + (1 + d) * NP + a;
                if (A.mode == 0) {
                  const R rs = fma(A.rk_a, ld<R>(eb + (C::O_RS + (1 + d) * NP + a) * RB), A.dt * ru[d]);
                  A.res[gi] = rs;
                  A.Qout[gi] = fma(A.rk_b, rs, ld<R>(eb + (C::O_Q + (1 + d) * NP + a) * RB));
                } else {
                  A.Qout[gi] = ru[d];
                }
              }
            }
          }
        }
      }
      __syncthreads();
    }

    // ---- F-I: WADG multiply + telescoping projection of r_p
    wadg_phases<C, R>(gb, q, A);
    constexpr int RES = wadg_result<C>();

    // ---- J: dp/dt = a!/N! b_N; outputs
    for (int a = q; a < NP; a += TG) {
      const R sc = __ldg(outN + a);
#pragma unroll
      for (int u = 0; u < ET; ++u) {
        const long long k = k0 + u;
        if (k >= A.elem_end) continue;
        const R dp = ld<R>(gb + u * EB + (RES + a) * RB) * sc;
        if (A.mode == 2) {
          A.Qout[k * NP + a] = dp;
        } else {
          const long long gi = k * 4 * NP + a;
          if (A.mode == 0) {
            const R rs = fma(A.rk_a, ld<R>(gb + u * EB + (C::O_RS + a) * RB), A.dt * dp);
            A.res[gi] = rs;
            A.Qout[gi] = fma(A.rk_b, rs, ld<R>(gb + u * EB + (C::O_Q + a) * RB));
          } else {
            A.Qout[gi] = dp;
          }
        }
      }
    }
    __syncthreads();
  }
}

// Halo pack: for each send face (local element k, face f) write the 4 own traces in the
// sender's canonical face ordering: buf[slot][c][i] = Q[k][c][fnode[f][i]].
template <int N, typename R>
__global__ void pack_kernel(const R* __restrict__ Q, const int* __restrict__ faces, int nfaces,
                            const uint16_t* __restrict__ fnode_bytes, R* __restrict__ buf) {
  constexpr int NP = cnp3(N), NFP = cnp2(N);
  const long long total = (long long)nfaces * 4 * NFP;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int slot = (int)(t / (4 * NFP));
    const int r = (int)(t - (long long)slot * 4 * NFP), c = r / NFP, i = r - c * NFP;
    const int k = faces[2 * slot], f = faces[2 * slot + 1];
    buf[t] = Q[(long long)k * 4 * NP + c * NP + __ldg(fnode_bytes + f * NFP + i) / (int)sizeof(R)];
  }
}

}  // namespace bbw
