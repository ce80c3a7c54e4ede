// Table layout of the 2D (triangle) path (R29-R30), shared by the host
// table builder (tables2d.cpp) and the 2D stage kernel (stage2d_kernel.cuh).  Compile-time offsets per
// (N, M, RB).  Canonical triangle order: rank2_n(a1, a2) = a2 (2n + 3 - a2)/2 + a1, a0 = n - a1 - a2.
// Edge f is opposite local vertex f, its vertices in increasing local index (0: (1,2), 1: (0,2), 2: (0,1));
// an edge coefficient is indexed by its exponent on the edge's SECOND vertex.
#pragma once
#include "layout.hpp"

namespace bbw {

__host__ __device__ constexpr int rank2c(int n, int a1, int a2) { return a2 * (2 * n + 3 - a2) / 2 + a1; }

struct Tab2Layout {
  int vg, ve, red, upw, lg, fnode, nbrvol, pdec;
  int s_invfacN, s_facN, s_outN, s_invfacM, s_post, s_invfacNm1, s_cfac, s_invf2, s_cf2;
  int total;
};

// VG  [Np2(N-1)]            ushort4: rank_N(b + e_j) * RB, j = 0..2        (gradient)
// VE  [Np2(N)]              ushort4: (rank_{N-1}(a - e_j) + 1) * RB or 0   (elevation, zero slot)
// RED [n=1..N+M][Np2(n-1)]  ushort4: rank_n(b + e_j) * RB                  (reductions n -> n-1)
// UPW [n=1..N][Np2(n)]      16 B: ushort4 (rank_{n-1}(a - e_j) + 1) * RB or 0, real 1/(a!)^2
// LG  [Np2(N)]              ushort4: byte offset of a in lift layer a_f of edge f (f = 0..2)
// FNODE  [3][N+1]           uint16: rank_N * RB of edge node i of edge f
// NBRVOL [3 f'][2 flip][N+1] uint16: rank_N of the neighbour's node matching own edge node i
// PDEC   [Np2(N+M)]         uint16: g1 | g2 << 8 of the degree-(N+M) coefficient g (product)
// scales: 1/a!, a!, a!/N! (deg N); 1/b! (deg M); (g!)^2 N!M!/(N+M)! (deg N+M); 1/b! (deg N-1);
//         c! and (c!)^2 (edge deg N); 1/(d!)^2 (edge deg N-1)
__host__ __device__ constexpr Tab2Layout tab2_layout(int N, int M, int RB) {
  Tab2Layout L{};
  int o = 0;
  L.vg = o;          o = al16(o + 8 * lnp2(N - 1));
  L.ve = o;          o = al16(o + 8 * lnp2(N));
  L.red = o;         o = al16(o + 8 * lnp3(N + M - 1));
  L.upw = o;         o = al16(o + 16 * (lnp3(N) - 1));
  L.lg = o;          o = al16(o + 8 * lnp2(N));
  L.fnode = o;       o = al16(o + 2 * 3 * (N + 1));
  L.nbrvol = o;      o = al16(o + 2 * 6 * (N + 1));
  L.pdec = o;        o = al16(o + 2 * lnp2(N + M));
  L.s_invfacN = o;   o = al16(o + RB * lnp2(N));
  L.s_facN = o;      o = al16(o + RB * lnp2(N));
  L.s_outN = o;      o = al16(o + RB * lnp2(N));
  L.s_invfacM = o;   o = al16(o + RB * lnp2(M));
  L.s_post = o;      o = al16(o + RB * lnp2(N + M));
  L.s_invfacNm1 = o; o = al16(o + RB * lnp2(N - 1));
  L.s_cfac = o;      o = al16(o + RB * (N + 1));
  L.s_invf2 = o;     o = al16(o + RB * N);
  L.s_cf2 = o;       o = al16(o + RB * (N + 1));
  L.total = o;
  return L;
}

// entry offsets of degree n inside RED (degrees 1..N+M) and UPW (degrees 1..N)
__host__ __device__ constexpr int red2_off(int n) { return lnp3(n - 2); }
__host__ __device__ constexpr int upw2_off(int n) { return lnp3(n - 1) - 1; }
// lift layer j (edge degree N-j, N-j+1 entries) inside one lift array
__host__ __device__ constexpr int lay2(int N, int j) { return j * (N + 1) - j * (j - 1) / 2; }

}  // namespace bbw
