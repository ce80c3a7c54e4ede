#include "mesh.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <sstream>

#include "tables.hpp"

namespace bbw {

std::string check_orientation(const GlobalMesh& g) {
  for (int64_t k = 0; k < g.K; ++k) {
    for (int v = 0; v < 4; ++v) {
      int64_t id = g.EV[4 * k + v];
      if (id < 0 || id >= g.nv) {
        std::ostringstream os;
        os << "element " << k << " references vertex " << id << " outside [0," << g.nv << ")";
        return os.str();
      }
    }
    const double* X0 = g.V + 3 * g.EV[4 * k];
    double e[3][3];
    for (int i = 0; i < 3; ++i)
      for (int d = 0; d < 3; ++d) e[i][d] = g.V[3 * g.EV[4 * k + i + 1] + d] - X0[d];
    double det = e[0][0] * (e[1][1] * e[2][2] - e[1][2] * e[2][1]) - e[0][1] * (e[1][0] * e[2][2] - e[1][2] * e[2][0]) +
                 e[0][2] * (e[1][0] * e[2][1] - e[1][1] * e[2][0]);
    if (!(det > 0)) {
      std::ostringstream os;
      os << "element " << k << " has non-positive Jacobian (det = " << det << "); vertices must be positively oriented";
      return os.str();
    }
  }
  return "";
}

void element_gradients(const GlobalMesh& g, int64_t k, double out[12]) {
  // x = X0 + sum_{i=1..3} l_i (X_i - X0)  =>  l_{1..3} = E^-1 (x - X0); grad l_0 = -sum grad l_i
  const double* X0 = g.V + 3 * g.EV[4 * k];
  double E[3][3];  // E[d][i] = (X_{i+1} - X0)_d
  for (int i = 0; i < 3; ++i)
    for (int d = 0; d < 3; ++d) E[d][i] = g.V[3 * g.EV[4 * k + i + 1] + d] - X0[d];
  double det = E[0][0] * (E[1][1] * E[2][2] - E[1][2] * E[2][1]) - E[0][1] * (E[1][0] * E[2][2] - E[1][2] * E[2][0]) +
               E[0][2] * (E[1][0] * E[2][1] - E[1][1] * E[2][0]);
  double inv[3][3];
  inv[0][0] = (E[1][1] * E[2][2] - E[1][2] * E[2][1]) / det;
  inv[0][1] = (E[0][2] * E[2][1] - E[0][1] * E[2][2]) / det;
  inv[0][2] = (E[0][1] * E[1][2] - E[0][2] * E[1][1]) / det;
  inv[1][0] = (E[1][2] * E[2][0] - E[1][0] * E[2][2]) / det;
  inv[1][1] = (E[0][0] * E[2][2] - E[0][2] * E[2][0]) / det;
  inv[1][2] = (E[0][2] * E[1][0] - E[0][0] * E[1][2]) / det;
  inv[2][0] = (E[1][0] * E[2][1] - E[1][1] * E[2][0]) / det;
  inv[2][1] = (E[0][1] * E[2][0] - E[0][0] * E[2][1]) / det;
  inv[2][2] = (E[0][0] * E[1][1] - E[0][1] * E[1][0]) / det;
  for (int d = 0; d < 3; ++d) {
    out[3 + d] = inv[0][d];
    out[6 + d] = inv[1][d];
    out[9 + d] = inv[2][d];
    out[d] = -(inv[0][d] + inv[1][d] + inv[2][d]);
  }
}

std::string build_connectivity(GlobalMesh& g) {
  const int64_t nf = 4 * g.K;
  g.etoe.assign(nf, -1);
  g.etof.assign(nf, -1);
  g.sigma.assign(nf, -1);
  // bucket faces by their smallest global vertex id (linear time, small buckets)
  auto key = [&](int64_t face, int64_t out[3]) {
    int64_t k = face / 4;
    int f = (int)(face % 4);
    for (int s = 0; s < 3; ++s) out[s] = g.EV[4 * k + FACE_V[f][s]];
    std::sort(out, out + 3);
  };
  std::vector<int64_t> cnt(g.nv + 1, 0);
  std::vector<int64_t> kmin(nf);
  for (int64_t face = 0; face < nf; ++face) {
    int64_t t[3];
    key(face, t);
    kmin[face] = t[0];
    cnt[t[0] + 1]++;
  }
  for (int64_t v = 0; v < g.nv; ++v) cnt[v + 1] += cnt[v];
  std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1), bucket(nf);
  for (int64_t face = 0; face < nf; ++face) bucket[pos[kmin[face]]++] = face;
  std::vector<std::pair<std::pair<int64_t, int64_t>, int64_t>> tmp;
  for (int64_t v = 0; v < g.nv; ++v) {
    tmp.clear();
    for (int64_t i = cnt[v]; i < cnt[v + 1]; ++i) {
      int64_t t[3];
      key(bucket[i], t);
      tmp.push_back({{t[1], t[2]}, bucket[i]});
    }
    std::sort(tmp.begin(), tmp.end());
    for (size_t i = 0; i + 1 < tmp.size(); ++i) {
      if (tmp[i].first != tmp[i + 1].first) continue;
      if (i + 2 < tmp.size() && tmp[i + 2].first == tmp[i].first) {
        std::ostringstream os;
        os << "face (" << v << "," << tmp[i].first.first << "," << tmp[i].first.second << ") is shared by more than two elements";
        return os.str();
      }
      int64_t a = tmp[i].second, b = tmp[i + 1].second;
      int64_t ka = a / 4, kb = b / 4;
      int fa = (int)(a % 4), fb = (int)(b % 4);
      g.etoe[a] = kb;
      g.etof[a] = (int8_t)fb;
      g.etoe[b] = ka;
      g.etof[b] = (int8_t)fa;
      for (int side = 0; side < 2; ++side) {
        int64_t k1 = side ? kb : ka, k2 = side ? ka : kb;
        int f1 = side ? fb : fa, f2 = side ? fa : fb;
        int64_t G[3], H[3];
        for (int s = 0; s < 3; ++s) {
          G[s] = g.EV[4 * k1 + FACE_V[f1][s]];
          H[s] = g.EV[4 * k2 + FACE_V[f2][s]];
        }
        int found = -1;
        for (int sg = 0; sg < 6 && found < 0; ++sg)
          if (G[0] == H[PERM[sg][0]] && G[1] == H[PERM[sg][1]] && G[2] == H[PERM[sg][2]]) found = sg;
        if (found < 0) return "internal error: face permutation not found";
        g.sigma[4 * k1 + f1] = (int8_t)found;
      }
      ++i;
    }
  }
  return "";
}

std::string partition(GlobalMesh& g, int nparts, const int cuts_in[3]) {
  g.owner.assign(g.K, 0);
  if (nparts <= 1) return "";
  int c[3] = {cuts_in ? cuts_in[0] : 0, cuts_in ? cuts_in[1] : 0, cuts_in ? cuts_in[2] : 0};
  if (c[0] <= 0 || c[1] <= 0 || c[2] <= 0) {
    // most cube-like factorisation px >= py >= pz
    int best = -1;
    for (int px = 1; px <= nparts; ++px)
      for (int py = 1; py <= px; ++py) {
        if (nparts % (px * py)) continue;
        int pz = nparts / (px * py);
        if (pz > py) continue;
        int score = px - pz;
        if (best < 0 || score < best) {
          best = score;
          c[0] = px;
          c[1] = py;
          c[2] = pz;
        }
      }
  }
  if (c[0] * c[1] * c[2] != nparts) return "partition cut counts do not multiply to world_size";
  std::vector<double> cen(3 * g.K);
  for (int64_t k = 0; k < g.K; ++k)
    for (int d = 0; d < 3; ++d) {
      double s = 0;
      for (int v = 0; v < 4; ++v) s += g.V[3 * g.EV[4 * k + v] + d];
      cen[3 * k + d] = s / 4;
    }
  std::vector<int64_t> idx(g.K);
  std::iota(idx.begin(), idx.end(), 0);
  // recursive: split range [lo,hi) along axis ax into c[ax] equal-count pieces
  struct Job { int64_t lo, hi; int ax, base, stride; };
  std::vector<Job> jobs{{0, g.K, 0, 0, c[1] * c[2]}};
  while (!jobs.empty()) {
    Job j = jobs.back();
    jobs.pop_back();
    std::stable_sort(idx.begin() + j.lo, idx.begin() + j.hi, [&](int64_t a, int64_t b) {
      return cen[3 * a + j.ax] < cen[3 * b + j.ax];
    });
    int n = c[j.ax];
    for (int p = 0; p < n; ++p) {
      int64_t lo = j.lo + (j.hi - j.lo) * p / n, hi = j.lo + (j.hi - j.lo) * (p + 1) / n;
      int base = j.base + p * j.stride;
      if (j.ax == 2) {
        for (int64_t i = lo; i < hi; ++i) g.owner[idx[i]] = base;
      } else {
        int nstride = (j.ax == 0) ? c[2] : 1;
        jobs.push_back({lo, hi, j.ax + 1, base, nstride});
      }
    }
  }
  return "";
}

Part build_part(const GlobalMesh& g, int rank, int nparts) {
  Part P;
  P.rank = rank;
  P.nparts = nparts;
  std::vector<int64_t> interior, boundary;
  for (int64_t k = 0; k < g.K; ++k) {
    if (g.owner[k] != rank) continue;
    bool bnd = false;
    for (int f = 0; f < 4; ++f) {
      int64_t nb = g.etoe[4 * k + f];
      if (nb >= 0 && g.owner[nb] != rank) bnd = true;
    }
    (bnd ? boundary : interior).push_back(k);
  }
  P.gid = interior;
  P.gid.insert(P.gid.end(), boundary.begin(), boundary.end());
  P.K_local = (int64_t)P.gid.size();
  P.n_interior = (int64_t)interior.size();
  std::vector<int32_t> g2l(g.K, -1);
  for (int64_t i = 0; i < P.K_local; ++i) g2l[P.gid[i]] = (int32_t)i;
  P.nbr.assign(4 * P.K_local, -1);
  P.code.assign(4 * P.K_local, 0);
  // shared faces per peer, in the canonical order (min global element id, that element's face)
  struct SF { int64_t key0; int key1; int32_t lk; int f; };
  std::vector<std::vector<SF>> shared(nparts);
  for (int64_t i = 0; i < P.K_local; ++i) {
    int64_t k = P.gid[i];
    for (int f = 0; f < 4; ++f) {
      int64_t nb = g.etoe[4 * k + f];
      int fp = g.etof[4 * k + f];
      if (nb < 0) continue;
      P.code[4 * i + f] = (uint8_t)(6 * fp + g.sigma[4 * k + f]);
      if (g.owner[nb] == rank) {
        P.nbr[4 * i + f] = g2l[nb];
      } else {
        SF s;
        s.key0 = std::min(k, nb);
        s.key1 = (k < nb) ? f : fp;
        s.lk = (int32_t)i;
        s.f = f;
        shared[g.owner[nb]].push_back(s);
      }
    }
  }
  // owner-local index of every element in its own partition (the same interior-first, global-id order
  // build_part gives that partition), for the peer-read transport's ghost map
  std::vector<int32_t> lidx(g.K, -1);
  {
    std::vector<uint8_t> isb(g.K, 0);
    for (int64_t k = 0; k < g.K; ++k)
      for (int f = 0; f < 4; ++f) {
        int64_t nb = g.etoe[4 * k + f];
        if (nb >= 0 && g.owner[nb] != g.owner[k]) isb[k] = 1;
      }
    std::vector<int32_t> nint(nparts, 0), cnt(nparts, 0);
    for (int64_t k = 0; k < g.K; ++k)
      if (!isb[k]) ++nint[g.owner[k]];
    for (int64_t k = 0; k < g.K; ++k)
      if (!isb[k]) lidx[k] = cnt[g.owner[k]]++;
    for (int r = 0; r < nparts; ++r) cnt[r] = nint[r];
    for (int64_t k = 0; k < g.K; ++k)
      if (isb[k]) lidx[k] = cnt[g.owner[k]]++;
  }
  P.send_off.assign(nparts + 1, 0);
  P.recv_off.assign(nparts + 1, 0);
  for (int r = 0; r < nparts; ++r) {
    auto& v = shared[r];
    std::sort(v.begin(), v.end(), [](const SF& a, const SF& b) {
      return a.key0 != b.key0 ? a.key0 < b.key0 : a.key1 < b.key1;
    });
    P.send_off[r + 1] = P.send_off[r] + (int64_t)v.size();
    P.recv_off[r + 1] = P.recv_off[r] + (int64_t)v.size();
    for (size_t j = 0; j < v.size(); ++j) {
      int64_t slot = P.recv_off[r] + (int64_t)j;
      P.nbr[4 * v[j].lk + v[j].f] = (int32_t)(-2 - slot);
      const int64_t nbg = g.etoe[4 * P.gid[v[j].lk] + v[j].f];
      P.gmap.push_back(r);
      P.gmap.push_back(lidx[nbg]);
      P.send_faces.push_back(v[j].lk);
      P.send_faces.push_back(v[j].f);
    }
  }
  return P;
}

}  // namespace bbw
