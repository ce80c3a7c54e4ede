// Host-side tables for the fast Bernstein path.  See tables.hpp for the formulas.
#include "tables.hpp"
#include "layout.hpp"

#include <cmath>
#include <cstring>

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
      W.u16x4(L.red, red_off(n) + (int)i, o);
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
        W.put<uint16_t>(L.lg + 16 * (int)i, f, (uint16_t)li);
        W.put<uint8_t>(L.lg + 16 * (int)i + 8, f, (uint8_t)j);
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
  // CSR of the Bernstein product (Eq. mcoeff): for g in degree N+M, all (a, b) with a + b = g
  {
    auto iN = indices3(N), iM = indices3(M), iH = indices3(N + M);
    int t = 0;
    for (size_t gi = 0; gi < iH.size(); ++gi) {
      W.put<int32_t>(L.csr_ptr, (int)gi, t);
      const int* g = iH[gi].a;
      for (size_t bi = 0; bi < iM.size(); ++bi) {
        const int* b = iM[bi].a;
        if (b[0] > g[0] || b[1] > g[1] || b[2] > g[2] || b[3] > g[3]) continue;
        int ar = rank3(N, g[1] - b[1], g[2] - b[2], g[3] - b[3]);
        W.put<uint32_t>(L.csr_terms, t++, (uint32_t)(ar * RB) | ((uint32_t)(bi * RB) << 16));
      }
    }
    W.put<int32_t>(L.csr_ptr, (int)iH.size(), t);
    if (t != lnp3(N) * lnp3(M)) throw std::runtime_error("CSR term count mismatch");
  }
  // ROWDEC: rows of degree N+M ordered by g2 + g3 (then g3), so that a warp pass of the
  // product takes rows of similar length
  {
    int r = 0;
    for (int s = 0; s <= N + M; ++s)
      for (int g3 = 0; g3 <= s; ++g3) {
        const int g2 = s - g3;
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
  auto c = projection_constants(N, M);
  for (int j = 0; j <= N; ++j) {
    T.cj[j] = c[j];
    T.gam[j] = (double)(lfact(j) * lfact(j) * (long double)c[N - j] / lfact(N + M));
    T.lam[j] = ((j & 1) ? -1.0 : 1.0) / (double)(j + 1);
  }
  return T;
}

}  // namespace bbw
