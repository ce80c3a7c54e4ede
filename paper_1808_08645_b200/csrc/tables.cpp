// Host-side tables for the fast Bernstein path.  See tables.hpp for the formulas.
#include "tables.hpp"

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
struct Blob {
  std::vector<uint8_t> b;
  size_t reserve(size_t bytes) {
    size_t off = (b.size() + 15) & ~size_t(15);
    b.resize(off + bytes, 0);
    return off;
  }
  template <class T>
  T* at(size_t off) { return reinterpret_cast<T*>(b.data() + off); }
};

long double prodfact(const int* a, int n) {
  long double p = 1.0L;
  for (int i = 0; i < n; ++i) p *= lfact(a[i]);
  return p;
}

template <class R>
void put_real(Blob& B, size_t off, int i, long double v) {
  R x = (R)v;
  std::memcpy(B.b.data() + off + i * sizeof(R), &x, sizeof(R));
}
}  // namespace

HostTables build_tables(int N, int M, int fp_bytes) {
  if (N < 1 || N > 9 || M < 0 || M > N) throw std::runtime_error("unsupported (N, M)");
  HostTables T;
  T.N = N;
  T.M = M;
  Blob B;
  const int NP = np3(N), NFP = np2(N), MP = np3(M), NPH = np3(N + M);

  // --- up[n][beta] (n = 0..N+M-1): ranks in degree n+1 of beta + e_j, exponents of beta
  T.off_up = B.reserve(sizeof(uint64_t) * np4(N + M - 1));
  for (int n = 0; n < N + M; ++n) {
    auto idx = indices3(n);
    uint64_t* dst = B.at<uint64_t>(T.off_up) + np4(n - 1);
    for (size_t i = 0; i < idx.size(); ++i) {
      const int* a = idx[i].a;
      int r[4] = {rank3(n + 1, a[1], a[2], a[3]), rank3(n + 1, a[1] + 1, a[2], a[3]),
                  rank3(n + 1, a[1], a[2] + 1, a[3]), rank3(n + 1, a[1], a[2], a[3] + 1)};
      dst[i] = pack_ranks4(r, a);
    }
  }
  // --- dn[n][alpha] (n = 0..N): ranks in degree n-1 of alpha - e_j (0 when alpha_j == 0)
  T.off_dn = B.reserve(sizeof(uint64_t) * np4(N));
  for (int n = 0; n <= N; ++n) {
    auto idx = indices3(n);
    uint64_t* dst = B.at<uint64_t>(T.off_dn) + np4(n - 1);
    for (size_t i = 0; i < idx.size(); ++i) {
      const int* a = idx[i].a;
      int r[4] = {0, 0, 0, 0};
      if (n > 0) {
        if (a[0] > 0) r[0] = rank3(n - 1, a[1], a[2], a[3]);
        if (a[1] > 0) r[1] = rank3(n - 1, a[1] - 1, a[2], a[3]);
        if (a[2] > 0) r[2] = rank3(n - 1, a[1], a[2] - 1, a[3]);
        if (a[3] > 0) r[3] = rank3(n - 1, a[1], a[2], a[3] - 1);
      }
      dst[i] = pack_ranks4(r, a);
    }
  }
  // --- dec[n][i] (n = 0..N+M): exponents packed 5 bits each
  T.off_dec = B.reserve(sizeof(uint32_t) * np4(N + M));
  for (int n = 0; n <= N + M; ++n) {
    auto idx = indices3(n);
    uint32_t* dst = B.at<uint32_t>(T.off_dec) + np4(n - 1);
    for (size_t i = 0; i < idx.size(); ++i) {
      const int* a = idx[i].a;
      dst[i] = (uint32_t)(a[0] | (a[1] << 5) | (a[2] << 10) | (a[3] << 15));
    }
  }
  // --- face tables
  auto tri = indices2(N);
  T.off_fnode = B.reserve(sizeof(uint16_t) * 4 * NFP);
  for (int f = 0; f < 4; ++f)
    for (int i = 0; i < NFP; ++i) {
      int a[4] = {0, 0, 0, 0};
      for (int s = 0; s < 3; ++s) a[FACE_V[f][s]] = tri[i].c[s];
      B.at<uint16_t>(T.off_fnode)[f * NFP + i] = (uint16_t)rank3(N, a[1], a[2], a[3]);
    }
  T.off_nbrvol = B.reserve(sizeof(uint16_t) * 24 * NFP);
  T.off_nbrface = B.reserve(sizeof(uint16_t) * 6 * NFP);
  for (int fp = 0; fp < 4; ++fp)
    for (int sg = 0; sg < 6; ++sg)
      for (int i = 0; i < NFP; ++i) {
        int d[3];
        for (int s = 0; s < 3; ++s) d[PERM[sg][s]] = tri[i].c[s];
        int a[4] = {0, 0, 0, 0};
        for (int t = 0; t < 3; ++t) a[FACE_V[fp][t]] = d[t];
        B.at<uint16_t>(T.off_nbrvol)[(fp * 6 + sg) * NFP + i] = (uint16_t)rank3(N, a[1], a[2], a[3]);
        if (fp == 0) B.at<uint16_t>(T.off_nbrface)[sg * NFP + i] = (uint16_t)rank2(N, d[1], d[2]);
      }
  // --- triangle reductions: triup[m][c] (m = 0..N-1): ranks in degree m+1 of c + e_s
  T.off_triup = B.reserve(sizeof(uint64_t) * np3(N - 1));
  for (int m = 0; m < N; ++m) {
    auto tm = indices2(m);
    uint64_t* dst = B.at<uint64_t>(T.off_triup) + np3(m - 1);
    for (size_t i = 0; i < tm.size(); ++i) {
      const int* c = tm[i].c;
      int r0 = rank2(m + 1, c[1], c[2]), r1 = rank2(m + 1, c[1] + 1, c[2]), r2 = rank2(m + 1, c[1], c[2] + 1);
      uint64_t v = (uint64_t)r0 | ((uint64_t)r1 << 8) | ((uint64_t)r2 << 16);
      v |= ((uint64_t)c[0] << 24) | ((uint64_t)c[1] << 29) | ((uint64_t)c[2] << 34);
      dst[i] = v;
    }
  }
  // --- L_0 7-point stencil on the face (degree N): neighbours c - e_a + e_b
  T.off_l0 = B.reserve(sizeof(uint64_t) * NFP);
  for (int i = 0; i < NFP; ++i) {
    const int* c = tri[i].c;
    uint64_t v = 0;
    for (int p = 0; p < 6; ++p) {
      int a = L0_PAIRS[p][0], b = L0_PAIRS[p][1];
      int nbi = i;
      if (c[a] > 0) {
        int d[3] = {c[0], c[1], c[2]};
        d[a] -= 1;
        d[b] += 1;
        nbi = rank2(N, d[1], d[2]);
      }
      v |= (uint64_t)nbi << (8 * p);
    }
    v |= ((uint64_t)c[0] << 48) | ((uint64_t)c[1] << 53) | ((uint64_t)c[2] << 58);
    B.at<uint64_t>(T.off_l0)[i] = v;
  }
  // --- lift gather: for volume alpha and face f, index into the (face, flux) layer buffer
  T.off_lgather = B.reserve(sizeof(uint32_t) * NP);
  {
    auto idx = indices3(N);
    for (int i = 0; i < NP; ++i) {
      const int* a = idx[i].a;
      uint32_t v = 0;
      for (int f = 0; f < 4; ++f) {
        int j = a[f];
        int off = 0;
        for (int jj = 0; jj < j; ++jj) off += np2(N - jj);
        int c[3];
        for (int s = 0; s < 3; ++s) c[s] = a[FACE_V[f][s]];
        int li = off + rank2(N - j, c[1], c[2]);
        v |= (uint32_t)li << (8 * f);
      }
      B.at<uint32_t>(T.off_lgather)[i] = v;
    }
  }
  // --- factorial scalings of the Bernstein product (Eq. mcoeff):
  //     h_g = [g! N! M!/(N+M)!] sum_b (r_{g-b}/(g-b)!) (c_b/b!)
  T.off_invfactN = B.reserve(fp_bytes * NP);
  T.off_invfactM = B.reserve(fp_bytes * MP);
  T.off_post = B.reserve(fp_bytes * NPH);
  {
    auto iN = indices3(N), iM = indices3(M), iH = indices3(N + M);
    const long double binv = lfact(N) * lfact(M) / lfact(N + M);
    for (int i = 0; i < NP; ++i) {
      long double v = 1.0L / prodfact(iN[i].a, 4);
      fp_bytes == 8 ? put_real<double>(B, T.off_invfactN, i, v) : put_real<float>(B, T.off_invfactN, i, v);
    }
    for (int i = 0; i < MP; ++i) {
      long double v = 1.0L / prodfact(iM[i].a, 4);
      fp_bytes == 8 ? put_real<double>(B, T.off_invfactM, i, v) : put_real<float>(B, T.off_invfactM, i, v);
    }
    for (int i = 0; i < NPH; ++i) {
      long double v = prodfact(iH[i].a, 4) * binv;
      fp_bytes == 8 ? put_real<double>(B, T.off_post, i, v) : put_real<float>(B, T.off_post, i, v);
    }
  }
  B.reserve(16);
  T.blob = std::move(B.b);

  auto c = projection_constants(N, M);
  for (int j = 0; j <= N; ++j) {
    T.cj[j] = c[j];
    // lift layer constants l_j = (-1)^j C(N,j)/(j+1)
    long double binom = lfact(N) / (lfact(j) * lfact(N - j));
    T.lj[j] = (double)(((j & 1) ? -1.0L : 1.0L) * binom / (long double)(j + 1));
  }
  return T;
}

}  // namespace bbw
