// far_tree.cuh — MIG repartitioning trees (Fig. 3) for the CUDA path.
//
// Written independently of oracle/ (no shared tables).  Node ids follow include/far.h.
// A node is packed into one 32-bit word so a lane can decode it from shared memory
// with one LDS regardless of which node it popped:
//   [0:3)   first hosted size index       (a node runs tasks of its own size;
//   [3:6)   second hosted size index (7=none)  the A100/H100 {S0..S3} node then runs size-3 tasks)
//   [6:9)   size index of the node itself (selects t_create / t_destroy, Table 2)
//   [9:13)  first child id  (15 = leaf)   — same first slice as the node
//   [13:17) second child id
//   [17:20) first slice of the second child
//   [20:24) first slice of the node (lo)
//   [24:28) number of slices of the node
//   [28:32) parent id (15 = root)
#pragma once
#include <cstdint>

namespace farb {

__host__ __device__ constexpr uint32_t pack_node(int lo, int sz, int c0, int c1, int szi, int ch1, int ch2, int ch2lo,
                                                 int par) {
  return (uint32_t)c0 | ((uint32_t)c1 << 3) | ((uint32_t)szi << 6) | ((uint32_t)ch1 << 9) | ((uint32_t)ch2 << 13) |
         ((uint32_t)ch2lo << 17) | ((uint32_t)lo << 20) | ((uint32_t)sz << 24) | ((uint32_t)par << 28);
}

__host__ __device__ __forceinline__ int nd_c0(uint32_t w) { return w & 7; }
__host__ __device__ __forceinline__ int nd_c1(uint32_t w) { return (w >> 3) & 7; }
__host__ __device__ __forceinline__ int nd_szi(uint32_t w) { return (w >> 6) & 7; }
__host__ __device__ __forceinline__ int nd_ch1(uint32_t w) { return (w >> 9) & 15; }
__host__ __device__ __forceinline__ int nd_ch2(uint32_t w) { return (w >> 13) & 15; }
__host__ __device__ __forceinline__ int nd_ch2lo(uint32_t w) { return (w >> 17) & 7; }
__host__ __device__ __forceinline__ int nd_lo(uint32_t w) { return (w >> 20) & 15; }
__host__ __device__ __forceinline__ int nd_sz(uint32_t w) { return (w >> 24) & 15; }
__host__ __device__ __forceinline__ int nd_par(uint32_t w) { return (w >> 28) & 15; }

constexpr int NONE = 7, LEAF = 15, ROOTP = 15;

// Profile families: NC = |C_G| (3: A30; 5: A100/H100).
template <int NC> struct Tree;

// A30: 4 -> {2,2} -> four leaves.  Sizes {1,2,4} -> indices 0,1,2.
template <> struct Tree<3> {
  static constexpr int S = 4, NN = 7;
  static constexpr int size[3] = {1, 2, 4};
  static constexpr uint32_t node[7] = {
      pack_node(0, 4, 2, NONE, 2, 1, 2, 2, ROOTP),
      pack_node(0, 2, 1, NONE, 1, 3, 4, 1, 0),
      pack_node(2, 2, 1, NONE, 1, 5, 6, 3, 0),
      pack_node(0, 1, 0, NONE, 0, LEAF, LEAF, 0, 1),
      pack_node(1, 1, 0, NONE, 0, LEAF, LEAF, 0, 1),
      pack_node(2, 1, 0, NONE, 0, LEAF, LEAF, 0, 2),
      pack_node(3, 1, 0, NONE, 0, LEAF, LEAF, 0, 2),
  };
  static constexpr int leaf_of_slice[4] = {3, 4, 5, 6};
};

// A100/H100 (odd split: first child gets the extra slice):
// 7 -> {S0..S3}:4 hosting [4,3] and {S4..S6}:3; 4 -> {2,2}; 3 -> {S4,S5}:2 and {S6}:1;
// 2 -> 1+1.  Sizes {1,2,3,4,7} -> indices 0..4.
template <> struct Tree<5> {
  static constexpr int S = 7, NN = 13;
  static constexpr int size[5] = {1, 2, 3, 4, 7};
  static constexpr uint32_t node[13] = {
      pack_node(0, 7, 4, NONE, 4, 1, 2, 4, ROOTP),
      pack_node(0, 4, 3, 2, 3, 3, 4, 2, 0),
      pack_node(4, 3, 2, NONE, 2, 5, 6, 6, 0),
      pack_node(0, 2, 1, NONE, 1, 7, 8, 1, 1),
      pack_node(2, 2, 1, NONE, 1, 9, 10, 3, 1),
      pack_node(4, 2, 1, NONE, 1, 11, 12, 5, 2),
      pack_node(6, 1, 0, NONE, 0, LEAF, LEAF, 0, 2),
      pack_node(0, 1, 0, NONE, 0, LEAF, LEAF, 0, 3),
      pack_node(1, 1, 0, NONE, 0, LEAF, LEAF, 0, 3),
      pack_node(2, 1, 0, NONE, 0, LEAF, LEAF, 0, 4),
      pack_node(3, 1, 0, NONE, 0, LEAF, LEAF, 0, 4),
      pack_node(4, 1, 0, NONE, 0, LEAF, LEAF, 0, 5),
      pack_node(5, 1, 0, NONE, 0, LEAF, LEAF, 0, 5),
  };
  static constexpr int leaf_of_slice[7] = {7, 8, 9, 10, 11, 12, 6};
};

// Node word of node u as a constexpr function (folds to a constant when u is a compile-time
// index, e.g. inside an unrolled loop; the static arrays above are host-side tables).
template <int NC> __host__ __device__ constexpr uint32_t tree_node(int u) {
  return NC == 3
             ? (u == 0 ? pack_node(0, 4, 2, NONE, 2, 1, 2, 2, ROOTP)
                : u == 1 ? pack_node(0, 2, 1, NONE, 1, 3, 4, 1, 0)
                : u == 2 ? pack_node(2, 2, 1, NONE, 1, 5, 6, 3, 0)
                : pack_node(u - 3, 1, 0, NONE, 0, LEAF, LEAF, 0, u <= 4 ? 1 : 2))
             : (u == 0 ? pack_node(0, 7, 4, NONE, 4, 1, 2, 4, ROOTP)
                : u == 1 ? pack_node(0, 4, 3, 2, 3, 3, 4, 2, 0)
                : u == 2 ? pack_node(4, 3, 2, NONE, 2, 5, 6, 6, 0)
                : u == 3 ? pack_node(0, 2, 1, NONE, 1, 7, 8, 1, 1)
                : u == 4 ? pack_node(2, 2, 1, NONE, 1, 9, 10, 3, 1)
                : u == 5 ? pack_node(4, 2, 1, NONE, 1, 11, 12, 5, 2)
                : u == 6 ? pack_node(6, 1, 0, NONE, 0, LEAF, LEAF, 0, 2)
                : pack_node(u - 7, 1, 0, NONE, 0, LEAF, LEAF, 0, 3 + (u - 7) / 2));
}
// leaf node id of slice s (constexpr form of Tree<NC>::leaf_of_slice)
template <int NC> __host__ __device__ constexpr int tree_leaf(int s) {
  return NC == 3 ? 3 + s : (s < 6 ? 7 + s : 6);
}
// One 3-bit field (at bit `shift` of the node word) of every node, packed into a 64-bit word
// (13 x 3 = 39 bits): looking a field up by a dynamic node id is a funnel shift instead of a
// dependent shared-memory load on the Alg. 1 event chain.
template <int NC> __host__ __device__ constexpr unsigned long long node_field_tab(int shift) {
  unsigned long long t = 0;
  for (int v = 0; v < (NC == 3 ? 7 : 13); ++v) t |= (unsigned long long)((tree_node<NC>(v) >> shift) & 7u) << (3 * v);
  return t;
}
template <int NC> __device__ __forceinline__ int node_c0(int v) {
  constexpr unsigned long long T = node_field_tab<NC>(0);
  return (int)((T >> (3 * v)) & 7u);
}
template <int NC> __device__ __forceinline__ int node_c1(int v) {
  constexpr unsigned long long T = node_field_tab<NC>(3);
  return (int)((T >> (3 * v)) & 7u);
}
template <int NC> __device__ __forceinline__ int node_szi(int v) {
  constexpr unsigned long long T = node_field_tab<NC>(6);
  return (int)((T >> (3 * v)) & 7u);
}
static_assert(tree_node<3>(6) == Tree<3>::node[6] && tree_node<3>(3) == Tree<3>::node[3], "A30 node table");
static_assert(tree_node<5>(12) == Tree<5>::node[12] && tree_node<5>(9) == Tree<5>::node[9] &&
                  tree_node<5>(6) == Tree<5>::node[6] && tree_node<5>(2) == Tree<5>::node[2],
              "A100 node table");

}  // namespace farb
