// Host-side mesh processing: validation, face connectivity by global vertex ids,
// geometric factors, recursive-coordinate-bisection partitioning and halo lists.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace bbw {

struct GlobalMesh {
  int64_t K = 0, nv = 0;
  const double* V = nullptr;   // [nv][3]
  const int64_t* EV = nullptr; // [K][4]
  std::vector<int64_t> etoe;   // [K][4] neighbour element (-1 boundary)
  std::vector<int8_t> etof;    // [K][4] neighbour face
  std::vector<int8_t> sigma;   // [K][4] slot permutation id (own slot s <-> neighbour slot PERM[sigma][s])
  std::vector<int32_t> owner;  // [K] partition id
};

// Returns "" on success, else an error message.
std::string build_connectivity(GlobalMesh& g);
std::string check_orientation(const GlobalMesh& g);
// grad(lambda_i), i = 0..3, of element k: out[12].
void element_gradients(const GlobalMesh& g, int64_t k, double out[12]);
// Recursive coordinate bisection into px*py*pz equal-count blocks (x, then y, then z).
std::string partition(GlobalMesh& g, int nparts, const int cuts[3]);

struct Part {
  int rank = 0, nparts = 1;
  int64_t K_local = 0, n_interior = 0;
  std::vector<int64_t> gid;       // local -> global
  std::vector<int32_t> nbr;       // [K_local][4]: >=0 local, -1 boundary, <= -2 ghost slot (-2 - slot)
  std::vector<uint8_t> code;      // [K_local][4]: 6 f' + sigma
  std::vector<int32_t> send_faces;// [nsend][2] (local element, face), grouped by destination rank
  std::vector<int64_t> send_off;  // [nparts+1] face offsets per destination rank
  std::vector<int64_t> recv_off;  // [nparts+1] ghost-slot offsets per source rank
  std::vector<int32_t> gmap;      // [nghost][2]: (owner rank, owner-local element id) of each ghost slot
  int64_t num_ghost() const { return recv_off.empty() ? 0 : recv_off.back(); }
};

Part build_part(const GlobalMesh& g, int rank, int nparts);

}  // namespace bbw
