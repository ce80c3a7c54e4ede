// Table layout shared by the host table builder (tables.cpp) and the device kernel
// (stage_kernel.cuh).  All offsets are compile-time functions of (N, M, RB = sizeof(real)).
//
// Index relations use the canonical multi-index rank (R19)
//   rank_n(a1,a2,a3) = Np(n) - Np(n-a3) + a2 (2(n-a3) + 3 - a2)/2 + a1,
// and all stencil tables hold BYTE offsets relative to the array they index, so that the
// kernel adds the array base and the element stride as immediates.
//
// Factorial scalings: with x' = a! x the one-degree reduction
// (E^T v)_b = (1/n) sum_j (b_j+1) v_{b+e_j} becomes (1/n) sum_j v'_{b+e_j}; with x'' = x/a!
// the elevation (E w)_a = (1/n) sum_j a_j w_{a-e_j} becomes (1/n) sum_j w''_{a-e_j}.
#pragma once
#include <stdint.h>

#ifndef BBW_RED32
#define BBW_RED32 1  // reduction table RED packed to 4 B per output (offset of b+e0 plus two 8-bit deltas)
#endif

namespace bbw {

__host__ __device__ constexpr int lnp3(int n) { return n < 0 ? 0 : (n + 1) * (n + 2) * (n + 3) / 6; }
__host__ __device__ constexpr int lnp2(int n) { return n < 0 ? 0 : (n + 1) * (n + 2) / 2; }
__host__ __device__ constexpr int lnp4(int n) { return n < 0 ? 0 : (n + 1) * (n + 2) * (n + 3) * (n + 4) / 24; }
__host__ __device__ constexpr int al16(int x) { return (x + 15) & ~15; }

struct TabLayout {
  // byte offsets of the sections
  int vg, ve, red, upw, lg, trired, triele, fnode, nbrvol, nbrface, rowdec, padoff, rowlen;
  int shd, shu, sho, shw, shs;  // shell-order ("triple") tables of the WADG projection
  int s_invfacN, s_facN, s_invfac2N, s_outN, s_invfacM, s_post, s_invfacNm1, s_cfac, s_invf2, s_cf2, s_rowpost;
  int total;
};

// VG   [Np(N-1)]            ushort4: rank_N(b+e_i)*RB, i = 0..3           (volume gradient)
// VE   [Np(N)]              ushort4: (rank_{N-1}(a-e_j)+1)*RB or 0        (volume elevation, zero slot)
// RED  [n=1..N+M][Np(n-1)]  ushort4: rank_n(b+e_j)*RB                     (reductions n -> n-1)
// UPW  [n=1..N][Np(n)]      16 B: ushort4 (rank_{n-1}(a-e_j)+1)*RB or 0, real weight 1/(a!)^2
// LG   [Np(N)]              ushort4: byte offset of coefficient a in lift layer a_f of face f (0..3)
// TRIRED [m=0..N-1][Np2(m)] ushort4: trirank_{m+1}(c+e_s)*RB, s = 0..2      (face reductions)
// TRIELE [Np2(N)]           ushort4: (trirank_{N-1}(c-e_s)+1)*RB or 0     (face elevation)
// FNODE  [4][Np2(N)]        uint16: rank_N of face node i of face f, times RB
// NBRVOL [24][Np2(N)]       uint16: rank_N of the matching neighbour node (code = 6 f' + sigma)
// NBRFACE [6][Np2(N)]       uint16: neighbour face-local index (ghost traces)
// ROWDEC [Np2(N+M)]        uint32: rows (g2, g3) of degree N+M: g2 | g3 << 8 | rank_{N+M}(0,g2,g3) << 16
// PADOFF [Np(N)]           uint16: byte offset of a in the zero-padded row copy (row stride RS)
// ROWLEN [Np2(N)]          uint8: length N - a2 - a3 + 1 of row (a2, a3) of degree N
// scale arrays (reals): 1/a!, a!, 1/(a!)^2, a!/N! (deg N); 1/b! (deg M); (g!)^2 N! M!/(N+M)! (deg N+M);
//                       1/b! (deg N-1); c!, 1/(d!)^2 (deg N-1), (c!)^2 (face, deg N);
//                       ROWPOST [Np2(N+M)] N!M!/(N+M)! (g2!)^2 (g3!)^2 per product output row (ROWDEC order)
__host__ __device__ constexpr TabLayout tab_layout(int N, int M, int RB) {
  TabLayout L{};
  int o = 0;
  L.vg = o;       o = al16(o + 8 * lnp3(N - 1));
  L.ve = o;       o = al16(o + 8 * lnp3(N));
  L.red = o;      o = al16(o + 8 * lnp4(N + M - 1));
  L.upw = o;      o = al16(o + 16 * (lnp4(N) - 1));
  L.lg = o;       o = al16(o + 8 * lnp3(N));
  L.trired = o;   o = al16(o + 8 * lnp3(N - 1));
  L.triele = o;   o = al16(o + 8 * lnp2(N));
  L.fnode = o;    o = al16(o + 2 * 4 * lnp2(N));
  L.nbrvol = o;   o = al16(o + 2 * 24 * lnp2(N));
  L.nbrface = o;  o = al16(o + 2 * 6 * lnp2(N));
  L.rowdec = o;    o = al16(o + 4 * lnp2(N + M));
  L.padoff = o;    o = al16(o + 2 * lnp3(N));
  L.rowlen = o;    o = al16(o + lnp2(N));
  L.s_invfacN = o;  o = al16(o + RB * lnp3(N));
  L.s_facN = o;     o = al16(o + RB * lnp3(N));
  L.s_invfac2N = o; o = al16(o + RB * lnp3(N));
  L.s_outN = o;     o = al16(o + RB * lnp3(N));
  L.s_invfacM = o;  o = al16(o + RB * lnp3(M));
  L.s_post = o;     o = al16(o + RB * lnp3(N + M));
  L.s_invfacNm1 = o; o = al16(o + RB * lnp3(N - 1));
  L.s_cfac = o;     o = al16(o + RB * lnp2(N));
  L.s_invf2 = o;    o = al16(o + RB * lnp2(N - 1));
  L.s_cf2 = o;      o = al16(o + RB * lnp2(N));
  L.s_rowpost = o;  o = al16(o + RB * lnp2(N + M));
  L.shd = o;        o = al16(o + 4 * lnp3(N + M - 1 > N ? N + M - 1 : N));
  L.shu = o;        o = al16(o + 4 * lnp3(N));
  L.sho = o;        o = al16(o + 4 * lnp3(N));
  L.shw = o;        o = al16(o + RB * lnp3(N));
  L.shs = o;        o = al16(o + RB * lnp3(N));
  L.total = o;
  return L;
}

// Shell order ("triple" ownership of the WADG projection): the multi-indices t = (a1,a2,a3)
// of every degree n <= N+M are enumerated by d = |t| (shell), then a3, then a2:
//   f(t) = Np(d-1) + a3 (2d+3-a3)/2 + a2,
// the same index at EVERY degree (a0 = n - d is implied), so degree n is the prefix f < Np(n).
// SHD[f] = f(t+e1) | (d+2-a3) << 16                      (f(t+e2) = f(t+e1)+1, f(t+e3) = f(t+e1)+d+2-a3)
// SHU[f] = (f(t-e1)+1) | (f(t-e2)+1) << 8 | (f(t-e3)+1) << 16 | d << 24     (0: t-e_j does not exist)
// SHO[a] = shell index f of the canonical degree-N coefficient a;  SHW[f] = 1/(a1! a2! a3!)^2;
// SHS[f] = a!/N!, a0 = N - d
__host__ __device__ constexpr int shell_of(int f) {
  int d = 0;
  while (lnp3(d) <= f) ++d;
  return d;  // shell d: Np(d-1) <= f < Np(d)
}

// offset (in entries) of degree n inside RED (degrees 1..N+M) and UPW (degrees 1..N)
__host__ __device__ constexpr int red_off(int n) { return lnp4(n - 2); }
__host__ __device__ constexpr int upw_off(int n) { return lnp4(n - 1) - 1; }
__host__ __device__ constexpr int trired_off(int m) { return lnp3(m - 1); }
// layer j of the lift buffer starts at entry sum_{j' < j} Np2(N - j')
__host__ __device__ constexpr int layer_off(int N, int j) { return lnp3(N) - lnp3(N - j); }

}  // namespace bbw
