// Host-side operator tables of the fast Bernstein path (independent of oracle/).
//
// All index relations are derived from the canonical multi-index rank
//   rank_n(a1,a2,a3) = Np(n) - Np(n-a3) + a2 (2(n-a3) + 3 - a2)/2 + a1
// (loop order a3 > a2 > a1, R19) and its triangle analogue
//   trirank_m(c0,c1,c2) = c2 (2m + 3 - c2)/2 + c1.
// Scalar constants:
//   c_j   projection constants, Thm main, from the closed-form
//         Bernstein mass eigenvalues lambda^n_k = |T| (n!)^2 d! / ((n+k+d)! (n-k)!)
//         (R8): sum_{j<=N-k} c_j lambda^{N-j}_k = lambda^{N+M}_k, k = N..0.
//   l_j   lift layer constants (-1)^j C(N,j)/(j+1) (R9, factorised lift P:266-268).
#pragma once
#include <array>
#include <cstdint>
#include <stdexcept>
#include <vector>

namespace bbw {

constexpr int np3(int n) { return n < 0 ? 0 : (n + 1) * (n + 2) * (n + 3) / 6; }
constexpr int np2(int n) { return n < 0 ? 0 : (n + 1) * (n + 2) / 2; }
constexpr int np4(int n) { return n < 0 ? 0 : (n + 1) * (n + 2) * (n + 3) * (n + 4) / 24; }  // sum_{m<=n} np3(m)

inline int rank3(int n, int a1, int a2, int a3) {
  int m = n - a3;
  return np3(n) - np3(m) + a2 * (2 * m + 3 - a2) / 2 + a1;
}
inline int rank2(int m, int c1, int c2) { return c2 * (2 * m + 3 - c2) / 2 + c1; }

struct MI { int a[4]; };
inline std::vector<MI> indices3(int n) {
  std::vector<MI> out;
  for (int a3 = 0; a3 <= n; ++a3)
    for (int a2 = 0; a2 <= n - a3; ++a2)
      for (int a1 = 0; a1 <= n - a3 - a2; ++a1) out.push_back(MI{{n - a1 - a2 - a3, a1, a2, a3}});
  return out;
}
struct TI { int c[3]; };
inline std::vector<TI> indices2(int m) {
  std::vector<TI> out;
  for (int c2 = 0; c2 <= m; ++c2)
    for (int c1 = 0; c1 <= m - c2; ++c1) out.push_back(TI{{m - c1 - c2, c1, c2}});
  return out;
}

// The 6 permutations sigma of the 3 face slots: own slot s <-> neighbour slot PERM[sigma][s].
constexpr int PERM[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
// face f = face opposite local vertex f; its vertices in increasing order
constexpr int FACE_V[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
// L_0 off-diagonal pairs (a, b): neighbour c - e_a + e_b
constexpr int L0_PAIRS[6][2] = {{0, 1}, {0, 2}, {1, 0}, {1, 2}, {2, 0}, {2, 1}};

inline uint64_t pack_ranks4(const int r[4], const int e[4]) {
  uint64_t v = 0;
  for (int j = 0; j < 4; ++j) v |= (uint64_t)(r[j] & 0x7FF) << (11 * j);
  for (int j = 0; j < 4; ++j) v |= (uint64_t)(e[j] & 0x1F) << (44 + 5 * j);
  return v;
}

// Byte image of all tables for one (N, M, RB) in the layout of layout.hpp, plus the
// per-(N,M) scalar constants passed as kernel parameters.
struct HostTables {
  int N = 0, M = 0, RB = 8;
  std::vector<uint8_t> blob;
  std::array<double, 10> cj{};   // projection constants c_0..c_N (Thm main)
  std::array<double, 10> gam{};  // upward-sweep level constants (n!)^2 c_{N-n} / (N+M)!, n = 0..N
  std::array<double, 10> lam{};  // lift layer constants (-1)^j/(j+1)  (= l_j / C(N,j))
};

// c_j for P^{N+M}_N and for M^-1 of the reference tetrahedron.
std::vector<double> projection_constants(int N, int M);
std::vector<double> mass_inverse_constants(int N);

// Build every table for (N, M); RB = sizeof(real) of the device path.
HostTables build_tables(int N, int M, int RB);
// 2D (triangle) path (layout2d.hpp; R29-R30): tables and projection constants with d = 2.
HostTables build_tables_2d(int N, int M, int RB);
std::vector<double> projection_constants_2d(int N, int M);

}  // namespace bbw
