// Aggregated Hamming distance of one key code against the G query codes of a
// GQA group, without one POPC per (head, word).
//
// PAPER: Alg. 3 lines 10-11 "S <- bitcount(bitwise_xor(Q_H, K_H^cache))"
// and P:255 "aggregate the scores S for shared KVCache" (sum over the group).
//
// B200 formulation: for bit b let c_b = #{h : q_h[b] = 1}
// and w_b = G - 2 c_b.  Then  D(k) = sum_h popc(q_h ^ k) = C0 + sum_b k_b w_b
// with C0 = sum_b c_b; the weights are split into signed magnitude bit planes
// (one LOP3 per plane and word) and a carry-save (full-adder LOP3) tree
// compresses the weighted words before counting, so the POPC count is
// ~log2(G*rbits) instead of G*W (group_distance_sw below).
#pragma once
#include "hata_common.cuh"

namespace hata {

// popcount of W words (weight 1) via a carry-save tree.
template <int W>
__device__ __forceinline__ uint32_t popc_words(const uint32_t* m) {
  if constexpr (W == 1) {
    return __popc(m[0]);
  } else if constexpr (W == 2) {
    return __popc(m[0]) + __popc(m[1]);
  } else if constexpr (W == 4) {
    uint32_t s, c;
    full_add(m[0], m[1], m[2], s, c);
    uint32_t ones = s ^ m[3], c2 = s & m[3];
    uint32_t twos = c ^ c2, fours = c & c2;
    return __popc(ones) + 2u * __popc(twos) + 4u * __popc(fours);
  } else {
    static_assert(W == 8, "W in {1,2,4,8}");
    uint32_t sa, ca, sb, cb, sc, cc;
    full_add(m[0], m[1], m[2], sa, ca);
    full_add(m[3], m[4], m[5], sb, cb);
    full_add(sa, sb, m[6], sc, cc);
    uint32_t ones = sc ^ m[7], cd = sc & m[7];
    uint32_t t, f1;
    full_add(ca, cb, cc, t, f1);
    uint32_t twos = t ^ cd, f2 = t & cd;
    uint32_t fours = f1 ^ f2, eights = f1 & f2;
    return __popc(ones) + 2u * __popc(twos) + 4u * __popc(fours) + 8u * __popc(eights);
  }
}

// ---------------------------------------------------------------------------
// Signed-weight form (fewer weighted words than the (c, G - c) planes above).
// With w_b = G - 2 c_b:  D(k) = C0 + sum_b k_b w_b,  C0 = sum_b c_b.
// For even G every w_b is even: v_b = w_b >> s (s = 1 for even G, else 0).
// Split v_b by sign into magnitude planes P_j (v_b > 0, bit j of |v_b|) and
// N_j (v_b < 0, bit j of |v_b|).  Since popc(k & N) = popc(N) - popc(~k & N)
// and P_j, N_j are disjoint:
//   D(k) = K0 + 2^s * sum_j 2^j popc((k & P_j) | (~k & N_j)),
//   K0   = C0 - 2^s * sum_j 2^j popc(N_j),
// one LOP3 per (plane, word).  Planes per group template: |v| <= G/2 (even G)
// or G (odd G) over the G the template serves.
constexpr __host__ __device__ int sw_planes_for_group(int GT) {
  return GT <= 2 ? 1 : (GT <= 4 ? 2 : 3);
}

__device__ __forceinline__ uint32_t lop_sel(uint32_t k, uint32_t P, uint32_t N) {   // (k & P) | (~k & N)
  return lop_mux(k, P, N);
}

// Three groups of 4 words with weights 1, 2, 4 (rbits = 128): 5 POPCs.
__device__ __forceinline__ uint32_t csa3_w4(const uint32_t (&m)[3][4]) {
  uint32_t s0, c0;
  full_add(m[0][0], m[0][1], m[0][2], s0, c0);
  uint32_t l0 = s0 ^ m[0][3], c0b = s0 & m[0][3];
  uint32_t s1, c1, s1b, c1b;
  full_add(m[1][0], m[1][1], m[1][2], s1, c1);
  full_add(m[1][3], c0, c0b, s1b, c1b);
  uint32_t l1 = s1 ^ s1b, c1c = s1 & s1b;
  uint32_t s2, c2, s2b, c2b, l2, c2c;
  full_add(m[2][0], m[2][1], m[2][2], s2, c2);
  full_add(m[2][3], c1, c1b, s2b, c2b);
  full_add(s2, s2b, c1c, l2, c2c);
  uint32_t l3, l4;
  full_add(c2, c2b, c2c, l3, l4);
  return __popc(l0) + 2u * __popc(l1) + 4u * __popc(l2) + 8u * __popc(l3) + 16u * __popc(l4);
}

// One carry-save tree over three groups of 8 words with weights 1, 2, 4
// (rbits = 256): 6 weighted words, 6 POPCs instead of 12 (one tree per
// group); the carries of each level join the next level.
__device__ __forceinline__ uint32_t csa3_w8(const uint32_t (&m)[3][8]) {
  uint32_t c1[4], d[7], f[7], h[3];
  uint32_t s1, s2, s3, l0, l1, l2, l3, l4, l5;
  // level 0: 8 words of plane 0
  full_add(m[0][0], m[0][1], m[0][2], s1, c1[0]);
  full_add(m[0][3], m[0][4], m[0][5], s2, c1[1]);
  full_add(s1, s2, m[0][6], s3, c1[2]);
  l0 = s3 ^ m[0][7]; c1[3] = s3 & m[0][7];
  // level 1: 8 words of plane 1 + 4 carries
  uint32_t t1, t2, t3, t4, t5;
  full_add(m[1][0], m[1][1], m[1][2], t1, d[0]);
  full_add(m[1][3], m[1][4], m[1][5], t2, d[1]);
  full_add(m[1][6], m[1][7], c1[0], t3, d[2]);
  full_add(c1[1], c1[2], c1[3], t4, d[3]);
  full_add(t1, t2, t3, t5, d[4]);
  l1 = t5 ^ t4; d[5] = t5 & t4;
  // level 2: 8 words of plane 2 + 6 carries
  uint32_t u1, u2, u3, u4, u5, u6;
  full_add(m[2][0], m[2][1], m[2][2], u1, f[0]);
  full_add(m[2][3], m[2][4], m[2][5], u2, f[1]);
  full_add(m[2][6], m[2][7], d[0], u3, f[2]);
  full_add(d[1], d[2], d[3], u4, f[3]);
  full_add(d[4], d[5], u1, u5, f[4]);
  full_add(u2, u3, u4, u6, f[5]);
  l2 = u6 ^ u5; f[6] = u6 & u5;
  // level 3: 7 carries; level 4: 3; level 5: 1
  uint32_t g1, g2;
  full_add(f[0], f[1], f[2], g1, h[0]);
  full_add(f[3], f[4], f[5], g2, h[1]);
  full_add(g1, g2, f[6], l3, h[2]);
  full_add(h[0], h[1], h[2], l4, l5);
  return __popc(l0) + 2u * __popc(l1) + 4u * __popc(l2) + 8u * __popc(l3) + 16u * __popc(l4) + 32u * __popc(l5);
}

// T = sum_j 2^j popc(M_j) over the W words (D = K0 + (T << s)).
template <int W, int JP>
__device__ __forceinline__ uint32_t group_distance_sw(const uint32_t (&k)[W], const uint32_t (&P)[JP][W],
                                                      const uint32_t (&N)[JP][W]) {
  uint32_t m[JP][W];
#pragma unroll
  for (int j = 0; j < JP; ++j)
#pragma unroll
    for (int w = 0; w < W; ++w) m[j][w] = lop_sel(k[w], P[j][w], N[j][w]);
  if constexpr (W == 4 && JP == 2) {
    uint32_t s0, c0, s1, c1, l1, c2, l2, l3;
    full_add(m[0][0], m[0][1], m[0][2], s0, c0);
    const uint32_t l0 = s0 ^ m[0][3], c0b = s0 & m[0][3];        // weight 1 | carries weight 2
    full_add(m[1][0], m[1][1], m[1][2], s1, c1);
    const uint32_t t = s1 ^ m[1][3], c1b = s1 & m[1][3];         // weight 2 | carries weight 4
    full_add(c0, c0b, t, l1, c2);                                // weight 2 | weight 4
    full_add(c1, c1b, c2, l2, l3);                               // weight 4 | weight 8
    return __popc(l0) + 2u * __popc(l1) + 4u * __popc(l2) + 8u * __popc(l3);
  } else if constexpr (W == 4 && JP == 3) {
    return csa3_w4(m);
  } else if constexpr (W == 8 && JP == 3) {
    return csa3_w8(m);
  } else {
    uint32_t d = 0;
#pragma unroll
    for (int j = 0; j < JP; ++j) d += popc_words<W>(m[j]) << j;
    return d;
  }
}

// Odd G (the G = 5 template): w_b = G - 2 c_b is odd, w_b = 2 t_b + 1 with
// t_b = (G-1)/2 - c_b, |t_b| <= (G+1)/2 = 3 -> two magnitude planes of t plus
// the key's own bits:  D(k) = K0 + popc(k) + 2 sum_j 2^j popc((k & P_j) | (~k & N_j)),
// K0 = C0 - 2 sum_j 2^j popc(N_j).  The key words enter the tree with weight 1
// as they are (no select): 2W selects instead of 3W.
template <int W>
__device__ __forceinline__ uint32_t group_distance_odd(const uint32_t (&k)[W], const uint32_t (&P)[2][W],
                                                       const uint32_t (&N)[2][W]) {
  uint32_t m[3][W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    m[0][w] = k[w];
    m[1][w] = lop_sel(k[w], P[0][w], N[0][w]);
    m[2][w] = lop_sel(k[w], P[1][w], N[1][w]);
  }
  if constexpr (W == 8) {
    return csa3_w8(m);
  } else if constexpr (W == 4) {
    return csa3_w4(m);
  } else {
    uint32_t d = 0;
#pragma unroll
    for (int j = 0; j < 3; ++j) d += popc_words<W>(m[j]) << j;
    return d;
  }
}

}  // namespace hata
