// Host-side tables of the 2D (triangle) fast Bernstein path (layout2d.hpp; R29-R30).
// Projection constants from the closed-form Bernstein mass eigenvalues with d = 2:
//   lambda^n_k = |T| (n!)^2 2! / ((n+k+2)! (n-k)!),  sum_{j<=N-k} c_j lambda^{N-j}_k = lambda^{N+M}_k  (Thm main,
//   P:441-470, in 2D).  Lift layer constants l_j / C(N,j) = (-1)^j/(j+1) (the 3D factorisation with d = 2,
//   checked against the 2D oracle's dense lift).
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "layout2d.hpp"
#include "tables.hpp"

namespace bbw {

static long double lf2(int n) {
  long double f = 1.0L;
  for (int i = 2; i <= n; ++i) f *= (long double)i;
  return f;
}

static long double mass_eig2(int n, int k) { return lf2(n) * lf2(n) * 2.0L / (lf2(n + k + 2) * lf2(n - k)); }

std::vector<double> projection_constants_2d(int N, int M) {
  std::vector<long double> c(N + 1, 0.0L);
  for (int k = N; k >= 0; --k) {
    const int j0 = N - k;
    long double s = mass_eig2(N + M, k);
    for (int j = 0; j < j0; ++j) s -= c[j] * mass_eig2(N - j, k);
    c[j0] = s / mass_eig2(N - j0, k);
  }
  return std::vector<double>(c.begin(), c.end());
}

namespace {
struct I3 {
  int a[3];
};
std::vector<I3> idx2(int n) {
  std::vector<I3> out;
  for (int a2 = 0; a2 <= n; ++a2)
    for (int a1 = 0; a1 <= n - a2; ++a1) out.push_back(I3{{n - a1 - a2, a1, a2}});
  return out;
}
int rk(int n, const int* a) { return rank2c(n, a[1], a[2]); }
long double pf(const int* a, int n) {
  long double p = 1.0L;
  for (int i = 0; i < n; ++i) p *= lf2(a[i]);
  return p;
}
constexpr int EDGE_V[3][2] = {{1, 2}, {0, 2}, {0, 1}};
struct W2 {
  std::vector<uint8_t>& b;
  template <class T>
  void put(int off, int i, T v) { std::memcpy(b.data() + off + (size_t)i * sizeof(T), &v, sizeof(T)); }
  void real(int off, int i, long double v, int RB) {
    if (RB == 8) put<double>(off, i, (double)v);
    else put<float>(off, i, (float)v);
  }
  void u16x4(int off, int i, int o0, int o1, int o2) {
    const int o[4] = {o0, o1, o2, 0};
    for (int j = 0; j < 4; ++j) {
      if (o[j] < 0 || o[j] > 0xFFFF) throw std::runtime_error("2D table offset out of 16-bit range");
      put<uint16_t>(off, 4 * i + j, (uint16_t)o[j]);
    }
  }
};
}  // namespace

HostTables build_tables_2d(int N, int M, int RB) {
  if (N < 1 || N > 9 || M < 0 || M > N) throw std::runtime_error("unsupported (N, M)");
  HostTables T;
  T.N = N;
  T.M = M;
  T.RB = RB;
  const Tab2Layout L = tab2_layout(N, M, RB);
  T.blob.assign(L.total, 0);
  W2 W{T.blob};
  auto plus = [](const int* a, int j, int d) {
    I3 r{{a[0], a[1], a[2]}};
    r.a[j] += d;
    return r;
  };
  {  // VG: b in degree N-1 -> rank_N(b + e_j)
    auto I = idx2(N - 1);
    for (size_t i = 0; i < I.size(); ++i) {
      const int* a = I[i].a;
      W.u16x4(L.vg, (int)i, rk(N, plus(a, 0, 1).a) * RB, rk(N, plus(a, 1, 1).a) * RB, rk(N, plus(a, 2, 1).a) * RB);
    }
  }
  auto elev = [&](int n, const int* a, int o[3]) {
    for (int j = 0; j < 3; ++j) o[j] = a[j] > 0 ? (rk(n - 1, plus(a, j, -1).a) + 1) * RB : 0;
  };
  {  // VE
    auto I = idx2(N);
    for (size_t i = 0; i < I.size(); ++i) {
      int o[3];
      elev(N, I[i].a, o);
      W.u16x4(L.ve, (int)i, o[0], o[1], o[2]);
    }
  }
  for (int n = 1; n <= N + M; ++n) {  // RED
    auto I = idx2(n - 1);
    for (size_t i = 0; i < I.size(); ++i) {
      const int* a = I[i].a;
      W.u16x4(L.red, red2_off(n) + (int)i, rk(n, plus(a, 0, 1).a) * RB, rk(n, plus(a, 1, 1).a) * RB,
              rk(n, plus(a, 2, 1).a) * RB);
    }
  }
  for (int n = 1; n <= N; ++n) {  // UPW
    auto I = idx2(n);
    for (size_t i = 0; i < I.size(); ++i) {
      int o[3];
      elev(n, I[i].a, o);
      const int e = upw2_off(n) + (int)i;
      for (int j = 0; j < 3; ++j) W.put<uint16_t>(L.upw + 16 * e, j, (uint16_t)o[j]);
      const long double f = pf(I[i].a, 3);
      W.real(L.upw + 16 * e + 8, 0, 1.0L / (f * f), RB);
    }
  }
  {  // LG: coefficient a, edge f: layer a_f, index = exponent on the edge's second vertex
    auto I = idx2(N);
    for (size_t i = 0; i < I.size(); ++i) {
      const int* a = I[i].a;
      int o[3];
      for (int f = 0; f < 3; ++f) o[f] = (lay2(N, a[f]) + a[EDGE_V[f][1]]) * RB;
      W.u16x4(L.lg, (int)i, o[0], o[1], o[2]);
    }
  }
  for (int f = 0; f < 3; ++f)  // FNODE: edge node i = exponent i on the second vertex, N - i on the first
    for (int i = 0; i <= N; ++i) {
      int a[3] = {0, 0, 0};
      a[EDGE_V[f][0]] = N - i;
      a[EDGE_V[f][1]] = i;
      W.put<uint16_t>(L.fnode, f * (N + 1) + i, (uint16_t)(rk(N, a) * RB));
    }
  for (int fp = 0; fp < 3; ++fp)  // NBRVOL: code = 2 f' + flip (flip: the neighbour's edge runs the other way)
    for (int fl = 0; fl < 2; ++fl)
      for (int i = 0; i <= N; ++i) {
        const int j = fl ? N - i : i;  // neighbour's second-vertex exponent
        int a[3] = {0, 0, 0};
        a[EDGE_V[fp][0]] = N - j;
        a[EDGE_V[fp][1]] = j;
        W.put<uint16_t>(L.nbrvol, (2 * fp + fl) * (N + 1) + i, (uint16_t)rk(N, a));
      }
  {  // PDEC
    auto I = idx2(N + M);
    for (size_t i = 0; i < I.size(); ++i)
      W.put<uint16_t>(L.pdec, (int)i, (uint16_t)(I[i].a[1] | (I[i].a[2] << 8)));
  }
  {  // scales
    auto iN = idx2(N), iM = idx2(M), iH = idx2(N + M), iN1 = idx2(N - 1);
    const long double binv = lf2(N) * lf2(M) / lf2(N + M);
    for (size_t i = 0; i < iN.size(); ++i) {
      const long double f = pf(iN[i].a, 3);
      W.real(L.s_invfacN, (int)i, 1.0L / f, RB);
      W.real(L.s_facN, (int)i, f, RB);
      W.real(L.s_outN, (int)i, f / lf2(N), RB);
    }
    for (size_t i = 0; i < iM.size(); ++i) W.real(L.s_invfacM, (int)i, 1.0L / pf(iM[i].a, 3), RB);
    for (size_t i = 0; i < iH.size(); ++i) {
      const long double f = pf(iH[i].a, 3);
      W.real(L.s_post, (int)i, f * f * binv, RB);
    }
    for (size_t i = 0; i < iN1.size(); ++i) W.real(L.s_invfacNm1, (int)i, 1.0L / pf(iN1[i].a, 3), RB);
    for (int i = 0; i <= N; ++i) {
      const long double f = lf2(N - i) * lf2(i);
      W.real(L.s_cfac, i, f, RB);
      W.real(L.s_cf2, i, f * f, RB);
    }
    for (int i = 0; i < N; ++i) {
      const long double f = lf2(N - 1 - i) * lf2(i);
      W.real(L.s_invf2, i, 1.0L / (f * f), RB);
    }
  }
  auto c = projection_constants_2d(N, M);
  for (int j = 0; j <= N; ++j) {
    T.cj[j] = c[j];
    T.gam[j] = (double)(lf2(j) * lf2(j) * (long double)c[N - j] / lf2(N + M));
    T.lam[j] = ((j & 1) ? -1.0 : 1.0) / (double)(j + 1);
  }
  return T;
}

}  // namespace bbw
