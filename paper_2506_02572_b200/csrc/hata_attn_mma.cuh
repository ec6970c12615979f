// Gather-fused sparse attention on the tensor cores (bf16 K/V; mma.sync
// m16n8k16, fp32 accumulation).  Alg. 3 lines 14-17 with the
// gather fused into the attention: the selected K/V rows are staged
// in smem by cp.async and never materialised in HBM.
//
// Per batch of staged rows, warp w takes 16-row groups w, w + NW, ...:
//   S  = Q . K_g^T           Q: the G heads of the group as A (rows >= G zero)
//   online softmax per warp  (running max m, sum l per head, fp32)
//   O += P . V_g             P split into bf16 hi + lo (two MMAs) so that the
//                            probabilities keep ~16 mantissa bits (R14)
// Afterwards the warps' (m, l, O) are merged in fixed warp order into the
// CTA partial: m_s[h], l_s[h] and st.acc (the same layout attend_rows gives).
#pragma once
#include "hata_decode.cuh"

namespace hata {

template <int GT, int D_HEAD>
__device__ __forceinline__ void attend_rows_mma(const int32_t* rows, int Rr, const __nv_bfloat16* __restrict__ Kc,
                                                const __nv_bfloat16* __restrict__ Vc, RowMap rmap, const __nv_bfloat16* qb,
                                                int G, float scale, uint8_t* kvbuf, int rows_cap, int rowb,
                                                float* m_s, float* l_s, AttnState<GT, D_HEAD>& st,
                                                uint64_t* bar, uint64_t* bar2, int kvpair, unsigned long long* tr = nullptr,
                                                int tb = 16) {
  static_assert(GT <= 8, "heads per group <= 8");
  constexpr int CH = D_HEAD * 2 / 16;            // 16-byte chunks per row
  constexpr int KS = D_HEAD / 16;                // k-steps over the head dim
  constexpr int NT = D_HEAD / 8;                 // output column tiles
  constexpr int NSL = AttnState<GT, D_HEAD>::NSL;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  // kvpair: the cache stores a token's K and V rows adjacently (V = K + d,
  // row stride 2d): one 512-byte bulk copy per selected token lands [K|V]
  // in one padded smem slot -- half the TMA requests of separate caches
  if (kvpair) rowb = 2 * D_HEAD * 2 + DEC_ROW_PAD;
  uint8_t* Ks = kvbuf;
  uint8_t* Vs = kvpair ? kvbuf + D_HEAD * 2 : kvbuf + rows_cap * rowb;
  uint8_t* const Ks0 = Ks;
  uint8_t* const Vs0 = Vs;

  // Q as A fragments held in registers for the whole call, read once from the
  // bf16 rows as stored (qb: [G][D_HEAD] smem); heads >= G and rows 8..15 are zero
  uint32_t qa[KS][2];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    const uint32_t* x = reinterpret_cast<const uint32_t*>(qb + gid * D_HEAD + ks * 16 + 2 * tig);
    qa[ks][0] = gid < G ? x[0] : 0u;
    qa[ks][1] = gid < G ? x[4] : 0u;
  }
  float O[NT][4];
#pragma unroll
  for (int t = 0; t < NT; ++t) O[t][0] = O[t][1] = O[t][2] = O[t][3] = 0.f;
  float m_run = -INFINITY, l_run = 0.f;          // head gid, this warp
  bool active = false;

  // more rows than one staging area holds: two half-size buffers, the next
  // batch's gather in flight while the current one is on the tensor cores
  const bool dbl = Rr > rows_cap;
  const int rc = dbl ? rows_cap / 2 : rows_cap;                   // rows per batch
  constexpr uint32_t ROWBYTES = D_HEAD * 2;
  auto issue = [&](int r0, int j) {
    const int nb = min(rc, Rr - r0);
    uint8_t* Kj = Ks + j * rc * rowb;
    uint8_t* Vj = Vs + j * rc * rowb;
    if (tid == 0) mbar_arrive_expect_tx((j ? bar2 : bar), 2u * ROWBYTES * (uint32_t)nb);
    __syncthreads();
    // gather: one bulk copy per selected row (TMA engine, no per-16B requests
    // in the LSU); request i -> warp i % NW, lane i / NW: a warp issues its
    // bulk copies one lane after another, so spread them over all warps
    if (kvpair) {
      for (int i = lane * DEC_WARPS + warp; i < nb; i += DEC_THREADS)
        bulk_g2s(Kj + i * rowb, Kc + rmap(rows[r0 + i]), 2 * ROWBYTES, (j ? bar2 : bar));
    } else {
      for (int i = lane * DEC_WARPS + warp; i < 2 * nb; i += DEC_THREADS) {
        const int which = i >= nb, rr = i - (which ? nb : 0);
        const __nv_bfloat16* src = (which ? Vc : Kc) + rmap(rows[r0 + rr]);
        bulk_g2s((which ? Vj : Kj) + rr * rowb, src, ROWBYTES, (j ? bar2 : bar));
      }
    }
  };
  uint32_t bpar = 0;                              // phase bit per buffer
  __syncthreads();                                // the staging area is free
  HATA_TRACE_AT(tr, tb + 4);
  if (Rr > 0) issue(0, 0);
  HATA_TRACE_AT(tr, tb + 3);
  for (int r0 = 0, bi = 0; r0 < Rr; r0 += rc, ++bi) {
    const int j = bi & 1;
    const int nb = min(rc, Rr - r0);
    if (dbl && r0 + rc < Rr) issue(r0 + rc, j ^ 1);              // its buffer was consumed last iteration
    mbar_wait(j ? bar2 : bar, (bpar >> j) & 1u);
    bpar ^= 1u << j;
    if (r0 == 0) HATA_TRACE_AT(tr, tb);
    const uint8_t* Ks = Ks0 + j * rc * rowb;
    const uint8_t* Vs = Vs0 + j * rc * rowb;
    for (int g0 = warp * 16; g0 < nb; g0 += DEC_WARPS * 16) {
      active = true;
      // S = Q K^T for rows g0 .. g0+15 (two 8-row tiles)
      float S[2][4];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        S[t][0] = S[t][1] = S[t][2] = S[t][3] = 0.f;
        int row = g0 + 8 * t + gid;
        row = row < nb ? row : g0;                                   // padded rows: any valid data
        const uint8_t* kr = Ks + row * rowb + 4 * tig;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const uint32_t b0 = *reinterpret_cast<const uint32_t*>(kr + ks * 32);
          const uint32_t b1 = *reinterpret_cast<const uint32_t*>(kr + ks * 32 + 16);
          const uint32_t a[4] = {qa[ks][0], 0u, qa[ks][1], 0u};
          mma_bf16_16816(S[t], a, b0, b1);
        }
      }
      // head gid owns S[t][0..1] = rows g0 + 8t + 2tig, +1
      float z[4];
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int row = g0 + 8 * t + 2 * tig + c;
          z[2 * t + c] = row < nb ? S[t][c] * scale : -INFINITY;
        }
      float mx = fmaxf(fmaxf(z[0], z[1]), fmaxf(z[2], z[3]));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float mn = fmaxf(m_run, mx);
      const float corr = (m_run == -INFINITY) ? 0.f : expf(m_run - mn);
      float pz[4], ps = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) { pz[i] = expf(z[i] - mn); ps += pz[i]; }
      ps += __shfl_xor_sync(0xffffffffu, ps, 1);
      ps += __shfl_xor_sync(0xffffffffu, ps, 2);
      l_run = l_run * corr + ps;
      m_run = mn;
#pragma unroll
      for (int t = 0; t < NT; ++t) { O[t][0] *= corr; O[t][1] *= corr; O[t][2] *= corr; O[t][3] *= corr; }
      // P as the A fragment (k = the 16 rows): rows 0-7 carry bf16(p) of the
      // heads, rows 8-15 the residual p - bf16(p), so one MMA yields both
      // halves (c0,c1: hi, c2,c3: lo; summed at the end)
      uint32_t pa[4];
      {
        const __nv_bfloat162 h0 = __floats2bfloat162_rn(pz[0], pz[1]);
        const __nv_bfloat162 h2 = __floats2bfloat162_rn(pz[2], pz[3]);
        const float2 b0f = __bfloat1622float2(h0), b2f = __bfloat1622float2(h2);
        pa[0] = *reinterpret_cast<const uint32_t*>(&h0);
        pa[2] = *reinterpret_cast<const uint32_t*>(&h2);
        pa[1] = pack_bf16x2(pz[0] - b0f.x, pz[1] - b0f.y);
        pa[3] = pack_bf16x2(pz[2] - b2f.x, pz[3] - b2f.y);
      }
      // O += P V over the 16 rows; V rows via ldmatrix.trans (padded rows)
      int vrow = g0 + (lane & 15);
      vrow = vrow < nb ? vrow : g0;
      const uint8_t* vr = Vs + vrow * rowb;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        uint32_t b0, b1;
        ldsm_x2_trans(b0, b1, vr + t * 16);
        mma_bf16_16816(O[t], pa, b0, b1);
      }
    }
  }
  // merge the warps in fixed order: smem [warp][GT][D_HEAD + 2] over the K/V area
  __syncthreads();
  HATA_TRACE_AT(tr, tb + 1);
  float* wp = reinterpret_cast<float*>(kvbuf);
  const int PS = D_HEAD + 2;
  if (gid < G) {
    float* dst = wp + (warp * GT + gid) * PS;
    if (tig == 0) { dst[0] = active ? m_run : -INFINITY; dst[1] = active ? l_run : 0.f; }
#pragma unroll
    for (int t = 0; t < NT; ++t)                                    // hi + lo halves of P
      *reinterpret_cast<float2*>(dst + 2 + t * 8 + 2 * tig) = make_float2(O[t][0] + O[t][2], O[t][1] + O[t][3]);
  }
  // only the first nact warps ever held rows
  const int nact = min(DEC_WARPS, (min(Rr, rows_cap) + 15) / 16);
  float* wgt = wp + DEC_WARPS * GT * PS;                            // [DEC_WARPS][GT] merge weights
  __syncthreads();
  // per head: max over warps (one warp per head, lanes = warps)
  if (warp < G) {
    const float mw = lane < nact ? wp[(lane * GT + warp) * PS] : -INFINITY;
    float Mx = mw;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) Mx = fmaxf(Mx, __shfl_xor_sync(0xffffffffu, Mx, o));
    const float wv = (mw == -INFINITY) ? 0.f : expf(mw - Mx);
    const float lw = lane < nact ? wp[(lane * GT + warp) * PS + 1] * wv : 0.f;
    float L = lw;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
    if (lane < DEC_WARPS) wgt[lane * GT + warp] = wv;
    if (lane == 0) { m_s[warp] = Mx; l_s[warp] = L; }
  }
  __syncthreads();
  HATA_TRACE_AT(tr, 29);
#pragma unroll
  for (int s = 0; s < NSL; ++s) {
    const int sl = tid + s * DEC_THREADS;
    const int h = sl / (D_HEAD / 2), e2 = sl % (D_HEAD / 2);
    float a0 = 0.f, a1 = 0.f;
    if (h < G) {
#pragma unroll 4
      for (int w = 0; w < nact; ++w) {
        const float* src = wp + (w * GT + h) * PS;
        const float sc = wgt[w * GT + h];
        const float2 v = *reinterpret_cast<const float2*>(src + 2 + 2 * e2);
        a0 = fmaf(v.x, sc, a0);
        a1 = fmaf(v.y, sc, a1);
      }
    }
    st.acc[s][0] = a0;
    st.acc[s][1] = a1;
  }
  __syncthreads();
  HATA_TRACE_AT(tr, 30);
}

// ---------------------------------------------------------------------------
// Sequence-shard phase 3 (hata_shard_partial_attn): attention over a split of
// the rank's selected rows -> raw (m, l, acc) partials.
template <typename T, int GT, int D_HEAD>
__global__ void __launch_bounds__(DEC_THREADS, 1) hata_partial_attn_kernel(const __grid_constant__ PartialParams p) {
  extern __shared__ __align__(1024) uint8_t psm[];
  constexpr int EB = sizeof(T);
  constexpr int NSL = AttnState<GT, D_HEAD>::NSL;
  const int sp = blockIdx.x, u = blockIdx.y, b = u / p.Hkv, g = u % p.Hkv, G = p.G;
  const int tid = threadIdx.x;
  const int QS = dec_qstride(D_HEAD);
  const int rowb = D_HEAD * EB + DEC_ROW_PAD;
  uint8_t* kv = psm;                                                         // [2][rows_cap][rowb]
  float* sc = reinterpret_cast<float*>(psm + ((2 * p.rows_cap * rowb + 127) & ~127));   // [GT][rows_cap]
  float* qf = sc + GT * p.rows_cap;                                          // [GT][QS]
  float* fm = qf + GT * QS;                                                  // m, l, corr
  uint64_t* bars = reinterpret_cast<uint64_t*>(fm + 32);                     // 2 mbarriers (bf16 gather)
  T* qraw = reinterpret_cast<T*>(bars + 2);                                  // [GT][d] bf16 rows
  int32_t* rows = reinterpret_cast<int32_t*>(qraw + GT * D_HEAD);             // this CTA's rows
  const T* qg = reinterpret_cast<const T*>(p.q) + ((int64_t)b * p.Hq + (int64_t)g * G) * D_HEAD;
  for (int i = tid; i < G * D_HEAD; i += DEC_THREADS) {
    qf[(i / D_HEAD) * QS + i % D_HEAD] = Elem<T>::to_f(qg[i]);
    qraw[i] = qg[i];
  }
  // this split's share of the rank's selected rows (ascending, contiguous)
  const int cnt = p.own_cnt[u];
  const int r0 = (int)((int64_t)cnt * sp / p.splits), r1 = (int)((int64_t)cnt * (sp + 1) / p.splits);
  const int nr = r1 - r0;
  for (int i = tid; i < nr; i += DEC_THREADS) rows[i] = p.own_idx[(int64_t)u * p.k + r0 + i];
  if (tid == 0) { mbar_init(&bars[0], 1); mbar_init(&bars[1], 1); fence_mbar_init(); }
  __syncthreads();
  const T* Kb = reinterpret_cast<const T*>(p.K) + (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh;
  const T* Vb = reinterpret_cast<const T*>(p.V) + (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh;
  AttnState<GT, D_HEAD> st;
  float* m_s = fm;
  float* l_s = fm + 8;
  float* corr_s = fm + 16;
  if constexpr (EB == 2) {
    // tensor-core gather-attention (the decode kernel's phase 4)
    attend_rows_mma<GT, D_HEAD>(rows, nr, reinterpret_cast<const __nv_bfloat16*>(p.K),
                                reinterpret_cast<const __nv_bfloat16*>(p.V),
                                RowMap{nullptr, 0, 0, (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh, p.kv_st},
                                reinterpret_cast<const __nv_bfloat16*>(qraw), G, p.scale, kv, p.rows_cap, rowb, m_s,
                                l_s, st, &bars[0], &bars[1],
                                reinterpret_cast<const uint8_t*>(p.V) == reinterpret_cast<const uint8_t*>(p.K) + D_HEAD * EB &&
                                    p.kv_st == 2 * D_HEAD);
  } else {
    attend_rows<T, GT, D_HEAD>(rows, nr, Kb, Vb, p.kv_st, qf, G, p.scale, kv, sc, p.rows_cap, rowb, m_s, l_s,
                               corr_s, st);
  }
  const int PS = D_HEAD + 2;
  float* part = p.partial + (int64_t)sp * p.B * p.Hq * PS;
#pragma unroll
  for (int s = 0; s < NSL; ++s) {
    const int sl = tid + s * DEC_THREADS;
    const int h = sl / (D_HEAD / 2), e2 = sl % (D_HEAD / 2);
    if (h < G) {
      float* pr = part + ((int64_t)b * p.Hq + g * G + h) * PS;
      pr[2 + 2 * e2] = st.acc[s][0];
      pr[3 + 2 * e2] = st.acc[s][1];
    }
  }
  if (tid < G) {
    float* pr = part + ((int64_t)b * p.Hq + g * G + tid) * PS;
    pr[0] = nr > 0 ? m_s[tid] : -INFINITY;
    pr[1] = nr > 0 ? l_s[tid] : 0.f;
  }
}

}  // namespace hata
