// Fused 2D (triangle) BBWADG RK-stage kernel for sm_100a (R29-R30).
//
// The triangle analogue of stage_kernel.cuh: per element and LSRK stage, fields (p, u_x, u_y):
//   volume   r_p = -div u, r_u = -grad p: barycentric derivative at degree N-1 (3-point), elevation
//   surface  Eq. sdf fluxes on the 3 edges, lift L^f = E^f_L L_0 with the 1-D edge operators
//            L_0 = |grad l_f| [(2N+2) I + N^2 E E^T] and layers s_j = -j/(j+1) R(s_{j-1}) (R30)
//   WADG     h = r_p c^2_M (Bernstein product, Eq. mcoeff), M reductions, telescoping down / up
//            sweeps with the 2D projection constants (Eq. telescope); M = 0: constant c^2
//   LSRK     res = a_s res + dt rhs; Q_out = Q_in + b_s res
// Factorial-scaled unweighted sums as in 3D (layout.hpp).  Groups of TG lanes per element (sub-warp for
// N <= 4), CTAs of 128 threads, a persistent grid-stride loop; shared memory per element holds the stencil
// arrays, the WADG work region aliases the volume / surface region.  The LSRK state is read at the output
// (measured: holding it in registers from the element start costs 7-14 % at (7,4), (3,1), (9,2) in fp64 --
// 8 more registers, one CTA per SM less -- and gains 4 % in fp32 only).
#pragma once
#include "layout2d.hpp"
#include "stage_kernel.cuh"

namespace bbw {

template <typename R>
struct Stage2DArgs {
  const R* Qin;
  R* Qout;
  R* res;
  const R* c2;
  const R* geo;        // [K][6]: grad(lambda_0..2)
  const int* nbr;      // [K][3] (-1 boundary)
  const uint8_t* code; // [K][3] = 2 f' + flip
  const R* src;        // [K][NP] or null
  const uint8_t* tab;
  long long elem_begin, elem_end;
  R rk_a, rk_b, dt, src_amp, tau_p, tau_u;
  R gam[10];
  int mode;  // 0 LSRK stage, 1 dQ/dt into Qout, 2 WADG apply (Qin = r[K][NP] -> Qout[K][NP])
};

__host__ __device__ constexpr int tg2d(int N) { return N <= 2 ? 8 : N <= 4 ? 16 : 32; }

template <int N_, int M_, typename R>
struct Stage2DCfg {
  static constexpr int N = N_, M = M_;
  static constexpr int NP = lnp2(N), NPM1 = lnp2(N - 1), MP = lnp2(M), NPH = lnp2(N + M), NPH1 = lnp2(N + M - 1);
  static constexpr int NE = N + 1;  // edge nodes
  static constexpr int RB = (int)sizeof(R), VEC = 16 / RB;
  static constexpr int T = 128, TG = tg2d(N), G = T / TG, GPW = TG < 32 ? 32 / TG : 1;
  static constexpr int KO = (NP + TG - 1) / TG;
  // per-element layout (reals)
  static constexpr int O_GEO = 0;          // grad l (6), per edge (n_x, n_y, |grad l_f|) at 6 + 3 f; ints at 16
  static constexpr int O_C = 24, O_RP = O_C + MP;
  static constexpr int O_X = rup(O_RP + NP, VEC);
  static constexpr int X_Q = O_X, X_G = X_Q + 3 * NP, X_F = X_G + 3 * (NPM1 + 1), X_Y = X_F + 6 * NE;
  static constexpr int X_L = X_Y + 6 * NE;  // 6 arrays x NP (layers concatenated)
  static constexpr int VS_END = X_L + 6 * NP;
  static constexpr int W_H = O_X, W_P = W_H + NPH, LEVB = W_P + NPH1;
  static __host__ __device__ constexpr int lev(int n) { return LEVB + lnp3(n - 1) + n + 1; }
  static constexpr int W_END = LEVB + lnp3(N) + N + 1;
  static constexpr int PER_E = rup(cmax(VS_END, W_END), VEC);
  static constexpr int EB = PER_E * RB;
  static constexpr int SMEM_BYTES = G * EB;
};

template <class C, typename R>
__global__ void __launch_bounds__(C::T) stage2d_kernel(const Stage2DArgs<R> A) {
  constexpr int N = C::N, M = C::M, NP = C::NP, NPM1 = C::NPM1, MP = C::MP, NE = C::NE, RB = C::RB;
  constexpr int TG = C::TG, KO = C::KO;
  constexpr Tab2Layout L = tab2_layout(N, M, RB);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, grp = tid / TG, q = tid - grp * TG;
  char* gb = reinterpret_cast<char*>(smem_raw) + grp * C::EB;
  auto sync = [&]() {
    if constexpr (TG <= 32) __syncwarp();
  };
  const uint8_t* tab = A.tab;
  const R* invfacN = reinterpret_cast<const R*>(tab + L.s_invfacN);
  const R* facN = reinterpret_cast<const R*>(tab + L.s_facN);
  const R* outN = reinterpret_cast<const R*>(tab + L.s_outN);
  const R* invfacM = reinterpret_cast<const R*>(tab + L.s_invfacM);
  const R* post = reinterpret_cast<const R*>(tab + L.s_post);
  const uint16_t* fnode = reinterpret_cast<const uint16_t*>(tab + L.fnode);
  const uint16_t* nbrvol = reinterpret_cast<const uint16_t*>(tab + L.nbrvol);
  auto LD = [&](int off) { return ld<R>(gb + off * RB); };
  auto ST = [&](int off, R v) { st<R>(gb + off * RB, v); };

  const long long nelem = A.elem_end - A.elem_begin;
  const int gw = grp % C::GPW;
  for (long long bw = (long long)blockIdx.x * C::G + (grp - gw); bw < nelem; bw += (long long)gridDim.x * C::G) {
    const long long batch = bw + gw;
    const long long k = A.elem_begin + batch;
    const bool live = batch < nelem;
    R ru[2][KO];
    // ---- A: loads
    if (live) {
      if (A.mode == 2) {
        for (int t = q; t < NP; t += TG) ST(C::O_RP + t, A.Qin[k * NP + t] * __ldg(invfacN + t));
      } else {
        for (int t = q; t < 3 * NP; t += TG) ST(C::X_Q + t, __ldg(A.Qin + k * 3 * NP + t));
        if (q < 6) ST(C::O_GEO + q, __ldg(A.geo + k * 6 + q));
        if (q < 3) {
          reinterpret_cast<int*>(gb + 16 * RB)[q] = __ldg(A.nbr + k * 3 + q);
          reinterpret_cast<uint8_t*>(gb + 16 * RB + 12)[q] = __ldg(A.code + k * 3 + q);
        }
      }
      for (int t = q; t < MP; t += TG) ST(C::O_C + t, __ldg(A.c2 + k * MP + t) * __ldg(invfacM + t));
    }
    sync();
    if (A.mode != 2) {
      if (q < 3) {  // outward normal, |grad lambda_f|
        const R gx = LD(C::O_GEO + 2 * q), gy = LD(C::O_GEO + 2 * q + 1);
        const R gl = sqrt(gx * gx + gy * gy), il = R(1) / gl;
        ST(C::O_GEO + 6 + 3 * q, -gx * il);
        ST(C::O_GEO + 7 + 3 * q, -gy * il);
        ST(C::O_GEO + 8 + 3 * q, gl);
      }
      if (q < 3) ST(C::X_G + q * (NPM1 + 1), R(0));  // zero slots of G''
      if (q < 6) ST(C::X_Y + q * NE, R(0));          // zero slots of Y''
      sync();
      const int* nbs = reinterpret_cast<const int*>(gb + 16 * RB);
      const uint8_t* cds = reinterpret_cast<const uint8_t*>(gb + 16 * RB + 12);
      // ---- B1a: neighbour traces (p, u_x, u_y) of every edge node
      constexpr int NI = 3 * NE, K1 = (NI + TG - 1) / TG;
      R tn[K1][3];
#pragma unroll
      for (int kk = 0; kk < K1; ++kk) {
        const int t = q + TG * kk;
        tn[kk][0] = tn[kk][1] = tn[kk][2] = R(0);
        if (t < NI && live) {
          const int f = t / NE, i = t - f * NE;
          const int nb = nbs[f];
          if (nb >= 0) {
            const R* qn = A.Qin + (long long)nb * 3 * NP + __ldg(nbrvol + cds[f] * NE + i);
            tn[kk][0] = __ldg(qn);
            tn[kk][1] = __ldg(qn + NP);
            tn[kk][2] = __ldg(qn + 2 * NP);
          }
        }
      }
      // ---- B2: g''_b = sum_j grad(l_j) q_{b+e_j} / b!  (div u, d_x p, d_y p)
      {
        R lg[6];
#pragma unroll
        for (int w = 0; w < 6; ++w) lg[w] = LD(C::O_GEO + w);
        const ushort4* vg = reinterpret_cast<const ushort4*>(tab + L.vg);
        for (int b = q; b < NPM1; b += TG) {
          const ushort4 o = __ldg(vg + b);
          const int off[3] = {o.x, o.y, o.z};
          const R sc = __ldg(reinterpret_cast<const R*>(tab + L.s_invfacNm1) + b);
          R dv = R(0), gx = R(0), gy = R(0);
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const char* p = gb + C::X_Q * RB + off[j];
            const R pj = ld<R>(p);
            gx = fma(lg[2 * j], pj, gx);
            gy = fma(lg[2 * j + 1], pj, gy);
            dv = fma(lg[2 * j], ld<R>(p + NP * RB), dv);
            dv = fma(lg[2 * j + 1], ld<R>(p + 2 * NP * RB), dv);
          }
          ST(C::X_G + 1 + b, dv * sc);
          ST(C::X_G + (NPM1 + 1) + 1 + b, gx * sc);
          ST(C::X_G + 2 * (NPM1 + 1) + 1 + b, gy * sc);
        }
      }
      // ---- B1b: fluxes F' = |grad l_f| c! F (Eq. sdf; boundary p+ = -p, u+ = u)
#pragma unroll
      for (int kk = 0; kk < K1; ++kk) {
        const int t = q + TG * kk;
        if (t < NI) {
          const int f = t / NE, i = t - f * NE;
          const int own = __ldg(fnode + f * NE + i);
          const char* eq = gb + C::X_Q * RB + own;
          const R pm = ld<R>(eq), uxm = ld<R>(eq + NP * RB), uym = ld<R>(eq + 2 * NP * RB);
          const bool bnd = nbs[f] < 0;
          const R pp = bnd ? -pm : tn[kk][0], uxp = bnd ? uxm : tn[kk][1], uyp = bnd ? uym : tn[kk][2];
          const R nx = LD(C::O_GEO + 6 + 3 * f), ny = LD(C::O_GEO + 7 + 3 * f);
          const R sc = LD(C::O_GEO + 8 + 3 * f) * __ldg(reinterpret_cast<const R*>(tab + L.s_cfac) + i);
          const R jp = pp - pm, jun = nx * (uxp - uxm) + ny * (uyp - uym);
          ST(C::X_F + (2 * f) * NE + i, R(0.5) * sc * (A.tau_p * jp - jun));
          ST(C::X_F + (2 * f + 1) * NE + i, R(0.5) * sc * (A.tau_u * jun - jp));
        }
      }
      sync();
      // ---- C1: r''_c[a] = -sum_j g''_c[a - e_j]
      {
        const ushort4* ve = reinterpret_cast<const ushort4*>(tab + L.ve);
#pragma unroll
        for (int kk = 0; kk < KO; ++kk) {
          const int a = q + TG * kk;
          ru[0][kk] = ru[1][kk] = R(0);
          if (a < NP) {
            const ushort4 o = __ldg(ve + a);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              const char* base = gb + (C::X_G + c * (NPM1 + 1)) * RB;
              const R v = ld<R>(base + o.x) + ld<R>(base + o.y) + ld<R>(base + o.z);
              if (c == 0) ST(C::O_RP + a, -v);
              else ru[c - 1][kk] = -v;
            }
          }
        }
      }
      // ---- C2: Y''[ff][d] = (F'[ff][d] + F'[ff][d+1]) / (d!)^2, edge degree N-1
      {
        const R* invf2 = reinterpret_cast<const R*>(tab + L.s_invf2);
        for (int t = q; t < 6 * N; t += TG) {
          const int ff = t / N, d = t - ff * N;
          ST(C::X_Y + ff * NE + 1 + d, (LD(C::X_F + ff * NE + d) + LD(C::X_F + ff * NE + d + 1)) * __ldg(invf2 + d));
        }
      }
      sync();
      // ---- C3: layer 0, w'_0[c] = (2N+2) F'[c] + (c!)^2 (Y''[c - e_0] + Y''[c - e_1])
      {
        const R* cf2 = reinterpret_cast<const R*>(tab + L.s_cf2);
        for (int t = q; t < 6 * NE; t += TG) {
          const int ff = t / NE, i = t - ff * NE;
          const R y = LD(C::X_Y + ff * NE + (i < N ? i + 1 : 0)) + LD(C::X_Y + ff * NE + i);
          ST(C::X_L + ff * NP + i, fma(__ldg(cf2 + i), y, R(2 * N + 2) * LD(C::X_F + ff * NE + i)));
        }
      }
      sync();
      // ---- D: lift layers j = 1..N, s_j[d] = -j/(j+1) (s_{j-1}[d] + s_{j-1}[d+1])
      static_for<1, N + 1, 1>([&](auto jc) {
        constexpr int j = decltype(jc)::value;
        constexpr int CNT = N - j + 1;
        constexpr R mu = R(-double(j) / double(j + 1));
        for (int t = q; t < 6 * CNT; t += TG) {
          const int ff = t / CNT, d = t - ff * CNT;
          const int src = C::X_L + ff * NP + lay2(N, j - 1) + d;
          ST(C::X_L + ff * NP + lay2(N, j) + d, mu * (LD(src) + LD(src + 1)));
        }
        sync();
      });
      // ---- E: gather the 3 edges' lifts; r''_p += S_p/(a!)^2 (+ source); r_u = a! r''_u + S_u/a!; LSRK u
      {
        const ushort4* lgt = reinterpret_cast<const ushort4*>(tab + L.lg);
        R nrm[6];
#pragma unroll
        for (int f = 0; f < 3; ++f) {
          nrm[2 * f] = LD(C::O_GEO + 6 + 3 * f);
          nrm[2 * f + 1] = LD(C::O_GEO + 7 + 3 * f);
        }
#pragma unroll
        for (int kk = 0; kk < KO; ++kk) {
          const int a = q + TG * kk;
          if (a < NP) {
            const ushort4 o = __ldg(lgt + a);
            const int lo[3] = {o.x, o.y, o.z};
            R sp = R(0), sx = R(0), sy = R(0);
#pragma unroll
            for (int f = 0; f < 3; ++f) {
              sp += ld<R>(gb + (C::X_L + 2 * f * NP) * RB + lo[f]);
              const R wu = ld<R>(gb + (C::X_L + (2 * f + 1) * NP) * RB + lo[f]);
              sx = fma(nrm[2 * f], wu, sx);
              sy = fma(nrm[2 * f + 1], wu, sy);
            }
            const R i1 = __ldg(invfacN + a), f1 = __ldg(facN + a);
            R rp = fma(sp, i1 * i1, LD(C::O_RP + a));
            if (A.src && live) rp = fma(A.src_amp * __ldg(A.src + k * NP + a), i1, rp);
            ST(C::O_RP + a, rp);
            const R r2[2] = {fma(ru[0][kk], f1, sx * i1), fma(ru[1][kk], f1, sy * i1)};
            if (live) {
#pragma unroll
              for (int d = 0; d < 2; ++d) {
                const long long gi = k * 3 * NP + (1 + d) * NP + a;
                if (A.mode == 0) {
                  const R r = fma(A.rk_a, __ldcs(A.res + gi), A.dt * r2[d]);
                  A.res[gi] = r;
                  A.Qout[gi] = fma(A.rk_b, r, __ldg(A.Qin + gi));
                } else {
                  A.Qout[gi] = r2[d];
                }
              }
            }
          }
        }
      }
      sync();
    }
    // ---- F-I: WADG of r''_p (Eq. mcoeff + Eq. telescope); M = 0: constant c^2
    R dp[KO];
    if constexpr (M == 0) {
      const R c0 = LD(C::O_C);
#pragma unroll
      for (int kk = 0; kk < KO; ++kk) {
        const int a = cmin(q + TG * kk, NP - 1);
        dp[kk] = c0 * __ldg(facN + a) * LD(C::O_RP + a);
      }
    } else {
      // F: h'_g = post_g sum_b r''_{g-b} c''_b, degree N+M output g owned per lane
      {
        const uint16_t* pdec = reinterpret_cast<const uint16_t*>(tab + L.pdec);
        for (int g = q; g < C::NPH; g += TG) {
          const int d = __ldg(pdec + g), g1 = d & 0xFF, g2 = d >> 8, g0 = N + M - g1 - g2;
          R acc = R(0);
          static_for<0, M + 1, 1>([&](auto b2c) {
            constexpr int b2 = decltype(b2c)::value;
            static_for<0, M + 1 - b2, 1>([&](auto b1c) {
              constexpr int b1 = decltype(b1c)::value;
              constexpr int b0 = M - b1 - b2;
              const int a1 = g1 - b1, a2 = g2 - b2, a0 = g0 - b0;
              if (a1 >= 0 && a2 >= 0 && a0 >= 0)
                acc = fma(LD(C::O_RP + rank2c(N, a1, a2)), LD(C::O_C + rank2c(M, b1, b2)), acc);
            });
          });
          ST(C::W_H + g, acc * __ldg(post + g));
        }
      }
      sync();
      // G: M reductions N+M -> N (H <-> P; the last lands in level N)
      const ushort4* red = reinterpret_cast<const ushort4*>(tab + L.red);
      auto reduce = [&](int src, int dst, int n) {
        const int cnt = lnp2(n - 1);
        const ushort4* rt = red + red2_off(n);
        for (int b = q; b < cnt; b += TG) {
          const ushort4 o = __ldg(rt + b);
          const char* s = gb + src * RB;
          ST(dst + b, (ld<R>(s + o.x) + ld<R>(s + o.y)) + ld<R>(s + o.z));
        }
        sync();
      };
      static_for<N + M, N, -1>([&](auto nc) {
        constexpr int n = decltype(nc)::value;
        constexpr int kk = N + M - n;
        constexpr int SRC = (kk % 2 == 0) ? C::W_H : C::W_P;
        constexpr int DST = (n - 1 == N) ? C::lev(N) : ((kk % 2 == 0) ? C::W_P : C::W_H);
        reduce(SRC, DST, n);
      });
      if (q < N) ST(C::lev(q) - 1, R(0));  // zero slots in front of levels 0..N-1
      // H: downward reductions, levels kept
      static_for<N, 0, -1>([&](auto nc) {
        constexpr int n = decltype(nc)::value;
        reduce(C::lev(n), C::lev(n - 1), n);
      });
      // I: upward in place, b_n[a] = sum_j b_{n-1}[a - e_j] + gam_n u_n[a] / (a!)^2, b_0 = gam_0 u_0
      if (q == 0) ST(C::lev(0), A.gam[0] * LD(C::lev(0)));
      sync();
      static_for<1, N + 1, 1>([&](auto nc) {
        constexpr int n = decltype(nc)::value;
        const uint8_t* up = tab + L.upw + 16 * upw2_off(n);
        const char* bp = gb + (C::lev(n - 1) - 1) * RB;
        for (int a = q; a < lnp2(n); a += TG) {
          const ushort4 o = __ldg(reinterpret_cast<const ushort4*>(up + 16 * a));
          const R w = A.gam[n] * __ldg(reinterpret_cast<const R*>(up + 16 * a + 8));
          const R v = (ld<R>(bp + o.x) + ld<R>(bp + o.y)) + ld<R>(bp + o.z);
          ST(C::lev(n) + a, fma(w, LD(C::lev(n) + a), v));
        }
        sync();
      });
#pragma unroll
      for (int kk = 0; kk < KO; ++kk) {
        const int a = cmin(q + TG * kk, NP - 1);
        dp[kk] = LD(C::lev(N) + a) * __ldg(outN + a);
      }
    }
    // ---- J: outputs / LSRK of p
#pragma unroll
    for (int kk = 0; kk < KO; ++kk) {
      const int a = q + TG * kk;
      if (!live || a >= NP) continue;
      if (A.mode == 2) {
        A.Qout[k * NP + a] = dp[kk];
      } else {
        const long long gi = k * 3 * NP + a;
        if (A.mode == 0) {
          const R r = fma(A.rk_a, __ldcs(A.res + gi), A.dt * dp[kk]);
          A.res[gi] = r;
          A.Qout[gi] = fma(A.rk_b, r, __ldg(A.Qin + gi));
        } else {
          A.Qout[gi] = dp[kk];
        }
      }
    }
    sync();
  }
}

}  // namespace bbw
