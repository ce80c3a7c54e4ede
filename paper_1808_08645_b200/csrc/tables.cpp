// Host-side tables for the fast Bernstein path.  See tables.hpp for the formulas.
#include "tables.hpp"
#include "layout.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>

namespace bbw {

static long double lfact(int n) {
  long double f = 1.0L;
  for (int i = 2; i <= n; ++i) f *= (long double)i;
  return f;
}

// Distinct eigenvalues of the degree-n Bernstein mass matrix on a d=3 simplex
// of measure vol (R8): lambda^n_k = vol (n!)^2 3! / ((n+k+3)! (n-k)!).
static long double mass_eig(int n, int k, long double vol) {
  return vol * lfact(n) * lfact(n) * 6.0L / (lfact(n + k + 3) * lfact(n - k));
}

std::vector<double> projection_constants(int N, int M) {
  // Thm main: in the modal basis sum_j c_j E E^T (E^{N+M}_N)^T is diagonal with
  // entries sum_{j<=N-k} c_j lambda^{N-j}_k / lambda^{N+M}_k, which must equal 1.
  std::vector<long double> c(N + 1, 0.0L);
  for (int k = N; k >= 0; --k) {
    int j0 = N - k;
    long double s = mass_eig(N + M, k, 1.0L);
    for (int j = 0; j < j0; ++j) s -= c[j] * mass_eig(N - j, k, 1.0L);
    c[j0] = s / mass_eig(N - j0, k, 1.0L);
  }
  return std::vector<double>(c.begin(), c.end());
}

std::vector<double> mass_inverse_constants(int N) {
  // Thm bbmass: sum_{j<=N-k} c_j lambda^{N-j}_k = 1 on the reference tet (|T| = 4/3).
  std::vector<long double> c(N + 1, 0.0L);
  const long double vol = 4.0L / 3.0L;
  for (int k = N; k >= 0; --k) {
    int j0 = N - k;
    long double s = 1.0L;
    for (int j = 0; j < j0; ++j) s -= c[j] * mass_eig(N - j, k, vol);
    c[j0] = s / mass_eig(N - j0, k, vol);
  }
  return std::vector<double>(c.begin(), c.end());
}

namespace {
long double prodfact(const int* a, int n) {
  long double p = 1.0L;
  for (int i = 0; i < n; ++i) p *= lfact(a[i]);
  return p;
}
struct Writer {
  std::vector<uint8_t>& b;
  template <class T>
  void put(int off, int i, T v) { std::memcpy(b.data() + off + (size_t)i * sizeof(T), &v, sizeof(T)); }
  void real(int off, int i, long double v, int RB) {
    if (RB == 8) put<double>(off, i, (double)v);
    else put<float>(off, i, (float)v);
  }
  void u16x4(int off, int i, const int o[4]) {
    for (int j = 0; j < 4; ++j) {
      if (o[j] < 0 || o[j] > 0xFFFF) throw std::runtime_error("table offset out of 16-bit range");
      put<uint16_t>(off, 4 * i + j, (uint16_t)o[j]);
    }
  }
};
}  // namespace


// ---- product row order (ROWDEC).  Rows (g2, g3) of degree N+M are sorted by g2 + g3 (so one warp
// pass holds rows of similar length); inside each warp pass the lane order is
// then chosen to minimise shared-memory wavefronts of the pass's accesses under the bank model that
// reproduces ncu's counts (profiles/r1_v4_*): 16-B row loads per c''-row (8 lanes per wavefront,
// 16-B units mod 8) and the scaled output stores (8-B: 16 lanes per wavefront, units mod 16; 4-B: 32
// lanes, units mod 32).  Deterministic annealing (fixed seed); any order is correct.
namespace {
// cost of one quarter-warp (loads) or half-warp (stores): max over bank units of distinct addresses
inline int group_cost(const int* addr, int n, int mod) {
  int best = 0;
  for (int a = 0; a < n; ++a) {
    if (addr[a] < 0) continue;
    int c = 0;
    bool dup = false;
    for (int b = 0; b < a; ++b)
      if (addr[b] == addr[a]) { dup = true; break; }
    if (dup) continue;
    for (int b = 0; b < n; ++b) {
      if (addr[b] < 0 || addr[b] % mod != addr[a] % mod) continue;
      bool seen = false;
      for (int e = 0; e < b; ++e)
        if (addr[e] == addr[b]) { seen = true; break; }
      if (!seen) ++c;
    }
    best = std::max(best, c);
  }
  return best;
}

std::vector<std::pair<int, int>> product_row_order_uncached(int N, int M, int RB) {
  const int VEC = 16 / RB, RS0 = (N + 1 + VEC - 1) / VEC * VEC, RS = RS0 + ((RS0 / VEC) % 2 == 0 ? VEC : 0);
  const int NFP = (N + 1) * (N + 2) / 2, SL = RB == 8 ? 16 : 32, SMOD = RB == 8 ? 16 : 32;
  std::vector<std::pair<int, int>> G, Bs, out;
  for (int s = 0; s <= N + M; ++s)
    for (int g3 = 0; g3 <= s; ++g3) G.push_back({s - g3, g3});
  for (int b3 = 0; b3 <= M; ++b3)
    for (int b2 = 0; b2 <= M - b3; ++b2) Bs.push_back({b2, b3});
  const int NR = (int)G.size(), NB = (int)Bs.size();
  uint64_t st = 0x9E3779B97F4A7C15ull;
  auto rnd = [&]() { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return st; };
  for (int r0 = 0; r0 < NR; r0 += 32) {  // one warp pass (a TG = 64 group is two warps)
    int rr[32];
    for (int l = 0; l < 32; ++l) rr[l] = r0 + l < NR ? r0 + l : -1;
    int smin = 1 << 20;
    for (int l = 0; l < 32; ++l)
      if (rr[l] >= 0) smin = std::min(smin, G[rr[l]].first + G[rr[l]].second);
    // per row r (of this pass) and c''-row B: 16-B unit of its input row (-2: no lane; NFP row = zeros)
    std::vector<int> nvec(NB, 0);
    std::vector<char> anyv(NB, 0);
    auto unit = [&](int r, int b) {
      if (r < 0) return -1;
      const int a2 = G[r].first - Bs[b].first, a3 = G[r].second - Bs[b].second;
      const bool valid = a2 >= 0 && a3 >= 0 && a2 + a3 <= N;
      return (valid ? a3 * (2 * N + 3 - a3) / 2 + a2 : NFP) * RS / VEC;
    };
    for (int b = 0; b < NB; ++b) {
      for (int l = 0; l < 32; ++l) {
        if (rr[l] < 0) continue;
        const int a2 = G[rr[l]].first - Bs[b].first, a3 = G[rr[l]].second - Bs[b].second;
        if (a2 >= 0 && a3 >= 0 && a2 + a3 <= N) anyv[b] = 1;
      }
      const int lamax = std::min(N + 1, N + 1 - smin + Bs[b].first + Bs[b].second);
      nvec[b] = anyv[b] ? (lamax + VEC - 1) / VEC : 0;
    }
    // product v5 (stage_kernel.cuh): a lane loads only the vectors of ITS input row that exist (predicated
    // on its own row length), invalid lanes load nothing
    auto lenA = [&](int r, int b) {
      if (r < 0) return 0;
      const int a2 = G[r].first - Bs[b].first, a3 = G[r].second - Bs[b].second;
      return (a2 >= 0 && a3 >= 0 && a2 + a3 <= N) ? N + 1 - a2 - a3 : 0;
    };
    auto qcost = [&](int q0) {  // loads of lanes q0..q0+7 over every c''-row and vector
      int c = 0, ad[8], ln[8];
      for (int b = 0; b < NB; ++b) {
        if (!nvec[b]) continue;
        for (int l = 0; l < 8; ++l) {
          ad[l] = unit(rr[q0 + l], b);
          ln[l] = lenA(rr[q0 + l], b);
        }
        for (int v = 0; v < nvec[b]; ++v) {
          int av[8];
          for (int l = 0; l < 8; ++l) av[l] = (ad[l] < 0 || VEC * v >= ln[l]) ? -1 : ad[l] + v;
          c += group_cost(av, 8, 8);
        }
      }
      return c;
    };
    auto hcost = [&](int h0) {  // output stores of lanes h0..h0+SL-1 over every x
      int c = 0, ad[32];
      for (int x = 0; x <= N + M; ++x) {
        for (int l = 0; l < SL; ++l) {
          const int r = rr[h0 + l];
          ad[l] = (r < 0 || x >= N + M + 1 - G[r].first - G[r].second) ? -1 : rank3(N + M, 0, G[r].first, G[r].second) + x;
        }
        c += group_cost(ad, SL, SMOD);
      }
      return c;
    };
    int qc[4], hc[2], cur = 0;
    for (int g = 0; g < 4; ++g) cur += (qc[g] = qcost(8 * g));
    for (int g = 0; g < 32 / SL; ++g) cur += (hc[g] = hcost(SL * g));
    int best = cur, bestrr[32];
    std::copy(rr, rr + 32, bestrr);
    double T = 3.0;
    const int iters = NB > 20 ? 600 : 2000;
    for (int it = 0; it < iters; ++it) {
      const int i = (int)(rnd() % 32), j = (int)(rnd() % 32);
      if (i / 8 == j / 8 || (rr[i] < 0 && rr[j] < 0)) continue;  // same quarter: loads unchanged
      std::swap(rr[i], rr[j]);
      const int qi = qcost(8 * (i / 8)), qj = qcost(8 * (j / 8));
      const int hi = hcost(SL * (i / SL)), hj = (i / SL == j / SL) ? hi : hcost(SL * (j / SL));
      const int c = cur - qc[i / 8] - qc[j / 8] + qi + qj - hc[i / SL] + hi - (i / SL == j / SL ? 0 : hc[j / SL] - hj);
      if (c <= cur || (double)(rnd() % 1000000) / 1e6 < std::exp(-(c - cur) / T)) {
        cur = c;
        qc[i / 8] = qi;
        qc[j / 8] = qj;
        hc[i / SL] = hi;
        hc[j / SL] = hj;
        if (c < best) best = c, std::copy(rr, rr + 32, bestrr);
      } else {
        std::swap(rr[i], rr[j]);
      }
      T = std::max(0.05, T * 0.997);
    }
    for (int l = 0; l < 32; ++l)
      if (bestrr[l] >= 0) out.push_back(G[bestrr[l]]);
  }
  return out;
}

std::vector<std::pair<int, int>> product_row_order(int N, int M, int RB) {
  static std::mutex mu;
  static std::map<int, std::vector<std::pair<int, int>>> cache;
  std::lock_guard<std::mutex> lk(mu);
  const int key = (N * 16 + M) * 16 + RB;
  auto it = cache.find(key);
  if (it == cache.end()) it = cache.emplace(key, product_row_order_uncached(N, M, RB)).first;
  return it->second;
}
}  // namespace

HostTables build_tables(int N, int M, int RB) {
  if (N < 1 || N > 9 || M < 0 || M > N) throw std::runtime_error("unsupported (N, M)");
  HostTables T;
  T.N = N;
  T.M = M;
  T.RB = RB;
  const TabLayout L = tab_layout(N, M, RB);
  T.blob.assign(L.total, 0);
  Writer W{T.blob};
  const int NFP = np2(N);

  // VG: volume gradient, b in degree N-1 -> rank_N(b + e_i)
  {
    auto idx = indices3(N - 1);
    for (size_t i = 0; i < idx.size(); ++i) {
      const int* a = idx[i].a;
      int o[4] = {rank3(N, a[1], a[2], a[3]) * RB, rank3(N, a[1] + 1, a[2], a[3]) * RB,
                  rank3(N, a[1], a[2] + 1, a[3]) * RB, rank3(N, a[1], a[2], a[3] + 1) * RB};
      W.u16x4(L.vg, (int)i, o);
    }
  }
  // VE: volume elevation, a in degree N -> (rank_{N-1}(a - e_j) + 1) * RB, 0 = zero slot
  auto elev_offsets = [&](int n, const int* a, int o[4]) {
    int d[4][3] = {{a[1], a[2], a[3]}, {a[1] - 1, a[2], a[3]}, {a[1], a[2] - 1, a[3]}, {a[1], a[2], a[3] - 1}};
    for (int j = 0; j < 4; ++j) o[j] = a[j] > 0 ? (rank3(n - 1, d[j][0], d[j][1], d[j][2]) + 1) * RB : 0;
  };
  {
    auto idx = indices3(N);
    for (size_t i = 0; i < idx.size(); ++i) {
      int o[4];
      elev_offsets(N, idx[i].a, o);
      W.u16x4(L.ve, (int)i, o);
    }
  }
  // RED: degree n -> n-1, b in degree n-1 -> rank_n(b + e_j) * RB
  for (int n = 1; n <= N + M; ++n) {
    auto idx = indices3(n - 1);
    for (size_t i = 0; i < idx.size(); ++i) {
      const int* a = idx[i].a;
      int o[4] = {rank3(n, a[1], a[2], a[3]) * RB, rank3(n, a[1] + 1, a[2], a[3]) * RB,
                  rank3(n, a[1], a[2] + 1, a[3]) * RB, rank3(n, a[1], a[2], a[3] + 1) * RB};
#if BBW_RED32
      // packed: byte offset of b + e0 | (b + e2 - (b + e0)) << 16 | (b + e3 - (b + e0)) << 24, the deltas in reals
      // (b + e1 is always the next real of the same row); 4 B per output instead of 8
      const int dz = (o[2] - o[0]) / RB, dw = (o[3] - o[0]) / RB;
      if (o[1] != o[0] + RB || dz < 0 || dz > 255 || dw < 0 || dw > 255 || o[0] > 0xFFFF)
        throw std::runtime_error("RED32 packing out of range");
      W.put<uint32_t>(L.red, red_off(n) + (int)i, (uint32_t)o[0] | ((uint32_t)dz << 16) | ((uint32_t)dw << 24));
#else
      W.u16x4(L.red, red_off(n) + (int)i, o);
#endif
    }
  }
  // UPW: degree n-1 -> n elevation with level weight 1/(a!)^2 (16-byte entries)
  for (int n = 1; n <= N; ++n) {
    auto idx = indices3(n);
    for (size_t i = 0; i < idx.size(); ++i) {
      int o[4];
      elev_offsets(n, idx[i].a, o);
      const int e = upw_off(n) + (int)i;
      for (int j = 0; j < 4; ++j) W.put<uint16_t>(L.upw + 16 * e, j, (uint16_t)o[j]);
      long double f = prodfact(idx[i].a, 4);
      W.real(L.upw + 16 * e + 8, 0, 1.0L / (f * f), RB);
    }
  }
  // LG: lift gather, per volume node and face: byte offset of (layer a_f, face-restricted index)
  {
    auto idx = indices3(N);
    for (size_t i = 0; i < idx.size(); ++i) {
      const int* a = idx[i].a;
      for (int f = 0; f < 4; ++f) {
        int j = a[f];
        int c[3];
        for (int s = 0; s < 3; ++s) c[s] = a[FACE_V[f][s]];
        int li = (layer_off(N, j) + rank2(N - j, c[1], c[2])) * RB;
        if (li > 0xFFFF) throw std::runtime_error("lift offset overflow");
        W.put<uint16_t>(L.lg + 8 * (int)i, f, (uint16_t)li);
      }
    }
  }
  // TRIRED: face degree m+1 -> m, c in degree m -> trirank_{m+1}(c + e_s) * RB
  for (int m = 0; m < N; ++m) {
    auto tm = indices2(m);
    for (size_t i = 0; i < tm.size(); ++i) {
      const int* c = tm[i].c;
      int o[4] = {rank2(m + 1, c[1], c[2]) * RB, rank2(m + 1, c[1] + 1, c[2]) * RB, rank2(m + 1, c[1], c[2] + 1) * RB,
                  0};
      W.u16x4(L.trired, trired_off(m) + (int)i, o);
    }
  }
  // TRIELE: face degree N-1 -> N, c in degree N -> (trirank_{N-1}(c - e_s) + 1) * RB or 0
  auto tri = indices2(N);
  for (int i = 0; i < NFP; ++i) {
    const int* c = tri[i].c;
    int o[4] = {c[0] > 0 ? (rank2(N - 1, c[1], c[2]) + 1) * RB : 0,
                c[1] > 0 ? (rank2(N - 1, c[1] - 1, c[2]) + 1) * RB : 0,
                c[2] > 0 ? (rank2(N - 1, c[1], c[2] - 1) + 1) * RB : 0, 0};
    W.u16x4(L.triele, i, o);
  }
  // face node maps
  for (int f = 0; f < 4; ++f)
    for (int i = 0; i < NFP; ++i) {
      int a[4] = {0, 0, 0, 0};
      for (int s = 0; s < 3; ++s) a[FACE_V[f][s]] = tri[i].c[s];
      W.put<uint16_t>(L.fnode, f * NFP + i, (uint16_t)(rank3(N, a[1], a[2], a[3]) * RB));
    }
  for (int fp = 0; fp < 4; ++fp)
    for (int sg = 0; sg < 6; ++sg)
      for (int i = 0; i < NFP; ++i) {
        int d[3];
        for (int s = 0; s < 3; ++s) d[PERM[sg][s]] = tri[i].c[s];
        int a[4] = {0, 0, 0, 0};
        for (int t = 0; t < 3; ++t) a[FACE_V[fp][t]] = d[t];
        W.put<uint16_t>(L.nbrvol, (fp * 6 + sg) * NFP + i, (uint16_t)rank3(N, a[1], a[2], a[3]));
        if (fp == 0) W.put<uint16_t>(L.nbrface, sg * NFP + i, (uint16_t)rank2(N, d[1], d[2]));
      }
  // ROWDEC / ROWPOST: rows of degree N+M in warp passes of similar g2 + g3, lane order chosen
  // against shared-memory bank conflicts (product_row_order)
  {
    int r = 0;
    for (const auto& gg : product_row_order(N, M, RB)) {
        const int g2 = gg.first, g3 = gg.second;
        const long double f = lfact(g2) * lfact(g3);
        W.real(L.s_rowpost, r, f * f * lfact(N) * lfact(M) / lfact(N + M), RB);
        W.put<uint32_t>(L.rowdec, r++, (uint32_t)g2 | ((uint32_t)g3 << 8) | ((uint32_t)rank3(N + M, 0, g2, g3) << 16));
      }
  }
  // PADOFF / ROWLEN: zero-padded row copy of degree-N arrays (row (a2,a3) at rowid*RS)
  {
    auto idx = indices3(N);
    for (size_t i = 0; i < idx.size(); ++i) {
      const int* a = idx[i].a;
      const int rowid = a[3] * (2 * N + 3 - a[3]) / 2 + a[2];
      const int VEC = 16 / RB, RS0 = (N + 1 + VEC - 1) / VEC * VEC;
      const int RS = RS0 + ((RS0 / VEC) % 2 == 0 ? VEC : 0);  // row stride (StageCfg::RS): odd # of 16-B vectors
      W.put<uint16_t>(L.padoff, (int)i, (uint16_t)((rowid * RS + a[1]) * RB));
    }
    int r = 0;
    for (int a3 = 0; a3 <= N; ++a3)
      for (int a2 = 0; a2 <= N - a3; ++a2) W.put<uint8_t>(L.rowlen, r++, (uint8_t)(N - a2 - a3 + 1));
  }
  // scale arrays
  {
    auto iN = indices3(N), iM = indices3(M), iH = indices3(N + M), iN1 = indices3(N - 1);
    const long double binv = lfact(N) * lfact(M) / lfact(N + M);
    for (int i = 0; i < (int)iN.size(); ++i) {
      long double f = prodfact(iN[i].a, 4);
      W.real(L.s_invfacN, i, 1.0L / f, RB);
      W.real(L.s_facN, i, f, RB);
      W.real(L.s_invfac2N, i, 1.0L / (f * f), RB);
      W.real(L.s_outN, i, f / lfact(N), RB);
    }
    for (int i = 0; i < (int)iM.size(); ++i) W.real(L.s_invfacM, i, 1.0L / prodfact(iM[i].a, 4), RB);
    for (int i = 0; i < (int)iH.size(); ++i) {
      long double f = prodfact(iH[i].a, 4);
      W.real(L.s_post, i, f * f * binv, RB);
    }
    for (int i = 0; i < (int)iN1.size(); ++i) W.real(L.s_invfacNm1, i, 1.0L / prodfact(iN1[i].a, 4), RB);
    auto t1 = indices2(N - 1);
    for (int i = 0; i < NFP; ++i) {
      long double f = prodfact(tri[i].c, 3);
      W.real(L.s_cfac, i, f, RB);
      W.real(L.s_cf2, i, f * f, RB);
    }
    for (int i = 0; i < (int)t1.size(); ++i) {
      long double f = prodfact(t1[i].c, 3);
      W.real(L.s_invf2, i, 1.0L / (f * f), RB);
    }
  }
  // shell-order tables (layout.hpp)
  {
    auto fsh = [](int a1, int a2, int a3) {
      const int d = a1 + a2 + a3;
      return np3(d - 1) + a3 * (2 * d + 3 - a3) / 2 + a2;
    };
    const int nd = std::max(N + M - 1, N);  // SHD up to degree N+M-1; SHU/SHO/SHW/SHS up to degree N
    for (int d = 0; d <= nd; ++d)
      for (int a3 = 0; a3 <= d; ++a3)
        for (int a2 = 0; a2 <= d - a3; ++a2) {
          const int a1 = d - a2 - a3, f = fsh(a1, a2, a3);
          const int f1 = fsh(a1 + 1, a2, a3);
          if (fsh(a1, a2 + 1, a3) != f1 + 1 || fsh(a1, a2, a3 + 1) != f1 + d + 2 - a3 || f1 > 0xFFFF)
            throw std::runtime_error("shell-order relation broken");
          W.put<uint32_t>(L.shd, f, (uint32_t)f1 | ((uint32_t)(d + 2 - a3) << 16));
          if (d <= N) {
            const int u1 = a1 > 0 ? fsh(a1 - 1, a2, a3) + 1 : 0, u2 = a2 > 0 ? fsh(a1, a2 - 1, a3) + 1 : 0,
                      u3 = a3 > 0 ? fsh(a1, a2, a3 - 1) + 1 : 0;
            if (u1 > 255 || u2 > 255 || u3 > 255) throw std::runtime_error("shell up offset overflow");
            W.put<uint32_t>(L.shu, f, (uint32_t)u1 | ((uint32_t)u2 << 8) | ((uint32_t)u3 << 16) | ((uint32_t)d << 24));
            W.put<uint32_t>(L.sho, rank3(N, a1, a2, a3), (uint32_t)f);  // canonical a -> shell index
            const long double g = lfact(a1) * lfact(a2) * lfact(a3);
            W.real(L.shw, f, 1.0L / (g * g), RB);
            W.real(L.shs, f, g * lfact(N - d) / lfact(N), RB);
          }
        }
  }
  auto c = projection_constants(N, M);
  for (int j = 0; j <= N; ++j) {
    T.cj[j] = c[j];
    T.gam[j] = (double)(lfact(j) * lfact(j) * (long double)c[N - j] / lfact(N + M));
    T.lam[j] = ((j & 1) ? -1.0 : 1.0) / (double)(j + 1);
  }
  return T;
}

}  // namespace bbw
