// Native face-topology builder (host code): SURVEY.md §8 (f1), the mesh half
// of the reference's builder (orodg/mesh.py:178-242, ForestMesh topology).
//
// Input: the Morton-sorted leaves (level, integer origin) of a forest over a
// root grid.  Output: the reference's face batches --
//   conforming per axis      (left, right), in leaf order of the left leaf;
//   hanging per (axis, orient) (coarse, fine, subface), sorted by (coarse,
//                              subface), one row per fine child;
//   boundary per (axis, side)  leaves in leaf order
// -- identical, array by array, to the vectorised numpy builder in mesh.py
// (tests/test_host_builders.py compares them on every fixture mesh).
//
// One open-addressing hash table over (level, origin) replaces the sorted
// code index; every leaf then looks across its 2d faces for the same-level
// neighbour, else the coarser parent (it is the fine side of a hanging face),
// else it checks that the finer child exists (it is the coarse side).  Any
// inconsistency (tiling gap, 2:1 violation, wrong subface count, origins
// beyond the key range) returns a non-zero code and the caller falls back to
// the numpy builder, which raises the reference's MeshError messages.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include "dg.h"

namespace {

struct Table {
  std::vector<uint64_t> keys;
  std::vector<int64_t> vals;
  uint64_t mask = 0;
  static uint64_t mix(uint64_t k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdULL;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ULL;
    k ^= k >> 33;
    return k;
  }
  void init(int64_t n) {
    uint64_t cap = 16;
    while (cap < (uint64_t)(2 * n + 1)) cap <<= 1;
    keys.assign(cap, ~0ULL);
    vals.assign(cap, -1);
    mask = cap - 1;
  }
  void put(uint64_t k, int64_t v) {
    uint64_t h = mix(k) & mask;
    while (keys[h] != ~0ULL) h = (h + 1) & mask;
    keys[h] = k;
    vals[h] = v;
  }
  int64_t get(uint64_t k) const {
    uint64_t h = mix(k) & mask;
    while (keys[h] != ~0ULL) {
      if (keys[h] == k) return vals[h];
      h = (h + 1) & mask;
    }
    return -1;
  }
};

constexpr int OBITS = 19;  // per-axis origin bits; 6 level bits above 3 x 19

inline uint64_t key_of(int dim, int64_t level, const int64_t* o) {
  uint64_t k = (uint64_t)level;
  for (int a = 0; a < dim; ++a) k = (k << OBITS) | (uint64_t)o[a];
  return k;
}

struct HangRow {
  int64_t coarse, fine, subface;
};

}  // namespace

struct dg_topo {
  int dim = 0;
  std::vector<int64_t> conf_l[3], conf_r[3];
  std::vector<HangRow> hang[6];   // (axis, orient) -> 2 * axis + orient
  std::vector<int64_t> bdry[6];   // (axis, side)
};

extern "C" {

int dg_topology_build(int dim, const int64_t* root_counts, const uint8_t* periodic, int64_t n,
                      const int64_t* levels, const int64_t* origins, dg_topo** out) {
  if (dim != 2 && dim != 3) return 2;
  int64_t max_level = 0;
  for (int64_t i = 0; i < n; ++i) max_level = std::max(max_level, levels[i]);
  if (max_level >= 40) return 2;
  for (int a = 0; a < dim; ++a)
    if (((root_counts[a] << (max_level + 1)) >> OBITS) != 0) return 2;  // key range
  Table T;
  T.init(n);
  for (int64_t i = 0; i < n; ++i) T.put(key_of(dim, levels[i], origins + i * dim), i);
  dg_topo* tp = new dg_topo;
  tp->dim = dim;
  const int n_sub = 1 << (dim - 1);
  int rc = 0;
  for (int64_t i = 0; i < n && rc == 0; ++i) {
    const int64_t L = levels[i];
    const int64_t* O = origins + i * dim;
    for (int axis = 0; axis < dim && rc == 0; ++axis) {
      for (int side = 0; side < 2; ++side) {
        int64_t nb[3];
        for (int a = 0; a < dim; ++a) nb[a] = O[a];
        nb[axis] += side ? 1 : -1;
        const int64_t count = root_counts[axis] << L;
        if (nb[axis] < 0 || nb[axis] >= count) {
          if (periodic[axis]) {
            nb[axis] = ((nb[axis] % count) + count) % count;
          } else {
            tp->bdry[2 * axis + side].push_back(i);
            continue;
          }
        }
        const int64_t j = T.get(key_of(dim, L, nb));
        if (j >= 0) {
          if (side == 1) {
            tp->conf_l[axis].push_back(i);
            tp->conf_r[axis].push_back(j);
          }
          continue;
        }
        int64_t jp = -1;
        int64_t pc[3];
        if (L > 0) {
          for (int a = 0; a < dim; ++a) pc[a] = nb[a] >> 1;
          jp = T.get(key_of(dim, L - 1, pc));
        }
        if (jp >= 0) {
          // this leaf is a fine child of a hanging face of leaf jp
          int64_t sf = 0;
          int k = 0;
          for (int fa = 0; fa < dim; ++fa) {
            if (fa == axis) continue;
            sf |= (O[fa] - 2 * pc[fa]) << k;
            ++k;
          }
          tp->hang[2 * axis + (1 - side)].push_back(HangRow{jp, i, sf});
          continue;
        }
        // the coarse side: its finer child across the face must exist
        int64_t ch[3];
        for (int a = 0; a < dim; ++a) ch[a] = 2 * nb[a];
        ch[axis] = 2 * nb[axis] + (side ? 0 : 1);
        if (T.get(key_of(dim, L + 1, ch)) < 0) {
          rc = 1;  // tiling gap or 2:1 violation: the numpy builder names it
          break;
        }
      }
    }
  }
  if (rc == 0) {
    for (int g = 0; g < 2 * dim && rc == 0; ++g) {
      auto& rows = tp->hang[g];
      std::stable_sort(rows.begin(), rows.end(), [](const HangRow& a, const HangRow& b) {
        return a.coarse != b.coarse ? a.coarse < b.coarse : a.subface < b.subface;
      });
      // every (coarse, axis, orient) group holds exactly 2^(d-1) subfaces
      size_t k = 0;
      while (k < rows.size()) {
        size_t e = k;
        while (e < rows.size() && rows[e].coarse == rows[k].coarse) ++e;
        if ((int)(e - k) != n_sub) {
          rc = 1;
          break;
        }
        k = e;
      }
    }
  }
  if (rc != 0) {
    delete tp;
    return rc;
  }
  *out = tp;
  return 0;
}

int dg_topology_counts(const dg_topo* tp, int64_t* n_conf, int64_t* n_hang, int64_t* n_bdry) {
  for (int a = 0; a < tp->dim; ++a) n_conf[a] = (int64_t)tp->conf_l[a].size();
  for (int g = 0; g < 2 * tp->dim; ++g) {
    n_hang[g] = (int64_t)tp->hang[g].size();
    n_bdry[g] = (int64_t)tp->bdry[g].size();
  }
  return 0;
}

int dg_topology_copy(const dg_topo* tp, int64_t* conf_left, int64_t* conf_right,
                     int64_t* hang_coarse, int64_t* hang_fine, int64_t* hang_subface,
                     int64_t* bdry_leaves) {
  size_t k = 0;
  for (int a = 0; a < tp->dim; ++a) {
    const size_t m = tp->conf_l[a].size();
    if (m) {
      std::memcpy(conf_left + k, tp->conf_l[a].data(), m * sizeof(int64_t));
      std::memcpy(conf_right + k, tp->conf_r[a].data(), m * sizeof(int64_t));
    }
    k += m;
  }
  k = 0;
  for (int g = 0; g < 2 * tp->dim; ++g)
    for (const HangRow& r : tp->hang[g]) {
      hang_coarse[k] = r.coarse;
      hang_fine[k] = r.fine;
      hang_subface[k] = r.subface;
      ++k;
    }
  k = 0;
  for (int g = 0; g < 2 * tp->dim; ++g) {
    const size_t m = tp->bdry[g].size();
    if (m) std::memcpy(bdry_leaves + k, tp->bdry[g].data(), m * sizeof(int64_t));
    k += m;
  }
  return 0;
}

int dg_topology_free(dg_topo* tp) {
  delete tp;
  return 0;
}

}  // extern "C"
