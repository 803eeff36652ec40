// Hermitian half spectrum (3-D, M = 16): node layout and phase generation helpers.
// Fragment of blfmm.cu (one translation unit): included inside
// namespace blfmm_gpu after the plan definition; not a standalone header.

// ------------------------------ Hermitian half spectrum (3-D, M = 16)
// Real weights make every expansion Hermitian in xi (V(-xi) = conj V(xi)),
// and every stage of the shared-grid sweep (P2M, M2M, couple, L2L, L2P) is
// diagonal in the quadrature node, so with T_i(m) the C-free product of the
// phase shifts and sums that reaches point i through node m,
//   u_i = w Re sum_m C_m T_i(m) = w Re sum_{m stored} Ct_m T_i(m),
// where Ct_m = C_m + C_m' if the mirror m' = M - m (per axis) of a stored node
// is a grid node that is not stored, and Ct_m = C_m otherwise. The grid
// -sigma + m dxi (m = 0..M-1) is symmetric except for its m_k = 0 endpoint,
// so the stored set is (e = index inside a box's expansion)
//   A  all rows (m1, m2), m3 in [8, 16)          2048 nodes  e = (16 m1 + m2) 8 + m3 - 8
//   C  the m3 = 0 plane                           256 nodes  e = 2048 + 16 m1 + m2
//   B  rows with m1 = 0 or m2 = 0, m3 in [1, 8)   217 nodes  e = 2304 + 7 rb + m3 - 1
// (2521 of 4096, padded to 2528 with zero nodes), and the missing nodes
// (m1, m2 >= 1, m3 in [1, 8)) are the mirrors of the A nodes with m1, m2 >= 1,
// m3 >= 9. P2M and L2P are the same DMMA GEMMs on the three blocks (62.5 % of
// the full tile work); M2M / couple index nodes through the node table.
// The imaginary part (max|Im|, mlfmm.cpp:343-358) of a mirrored pair is
// (C_m - C_m') Im T, not a function of Ct T: the spectral tables are cell
// averages over one-sided cells [xi_m, xi_m + dxi] and are not even (IMQ / MQ),
// so L2P carries a second GEMM on the A block with the stored locals scaled by
// D_e = (C_m - C_m') / Ct_m (D_e = 1 for nodes whose mirror is off the grid or
// stored); blocks B and C have D = 1.
constexpr int kH16A = 2048, kH16C = 256, kH16BR = 31, kH16B = kH16BR * 7;
constexpr int kH16K = kH16A + kH16C + kH16B;  // 2521
constexpr int kH16Ks = 2528;                  // padded: 32-byte aligned boxes
__host__ __device__ __forceinline__ void h16_brow(int rb, int& m1, int& m2) {
  m1 = rb < 16 ? 0 : rb - 15;
  m2 = rb < 16 ? rb : 0;
}

// (polar_small / gen_row16: k_expansions.inc.cuh, shared with the 2-D kernels)
struct LeafGeom {  // leaf centre from its Morton key (geometry.hpp:62-64)
  double lo[3], side[3];
  int L;
  __device__ __forceinline__ void centre(uint32_t key, double c[3]) const {
    int q[3];
    morton_decode<3>(key, L, q);
#pragma unroll
    for (int k = 0; k < 3; ++k) c[k] = lo[k] + (q[k] + 0.5) * side[k];
  }
};
