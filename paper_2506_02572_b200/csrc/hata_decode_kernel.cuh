// The fused HATA decode kernel (one launch per decode step).  Parameters,
// shared-memory layout and the attention helper live in hata_decode.cuh.
//
// Phases of one CTA (rank r of unit u = (b, KV head g)), DESIGN.md "Decode kernel":
//   0  start the bulk copies: W_g and this rank's whole code chunk (q-independent)
//   1  Encode & Cache update: hash the G query heads (+ the new key), write the
//      appended K/V/code rows                          Alg. 3 lines 2-9
//   2  Hamming score + GQA sum + D histogram          Alg. 3 lines 10-11
//   3  exact top-k' by counting select: one histogram exchange between the
//      unit's ranks, threshold + tie quotas, order-preserving compaction of
//      this rank's equal share of the selection        Alg. 3 lines 12-13
//   4  gather-fused softmax attention over that share Alg. 3 lines 14-17
//   5  rank-ordered flash-decoding merge by the last rank to finish
#pragma once
#include "hata_attn_mma.cuh"
#include "hata_decode.cuh"

namespace hata {

// Block-wide exclusive scan of one int per thread.  buf: >= DEC_WARPS + 1 ints
// of smem, not in use by anybody else across the call.
__device__ __forceinline__ int block_excl_scan(int v, int* buf, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  __syncthreads();
  if (lane == 31) buf[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const int w = lane < DEC_WARPS ? buf[lane] : 0;
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < DEC_WARPS) buf[lane] = wi - w;
    if (lane == DEC_WARPS - 1) buf[DEC_WARPS] = wi;
  }
  __syncthreads();
  total = buf[DEC_WARPS];
  return buf[warp] + inc - v;
}

// One rank's D array as seen by the selection scan.
struct ChunkRef {
  const uint16_t* D;   // 16-byte aligned
  int L;               // tokens
  int quota;           // ties (D == thr) selected from this chunk
  int base;            // selection position of its first selected token
  int fromg;           // D lives in global memory (L2): load with ld.cg
  int tok0;            // sequence index of its token 0
};

// 8-bit masks of (D < thr) and (D == thr) for tokens j .. j+7 of a chunk,
// tokens >= s1 masked out.
__device__ __forceinline__ void d_masks(const uint16_t* Dc, bool fromg, int j, int s1, int thr, uint32_t& ltm,
                                        uint32_t& tim) {
  uint32_t v[4];
  if (j + 8 <= s1) {
    const uint4 x = fromg ? __ldcg(reinterpret_cast<const uint4*>(Dc + j)) : *reinterpret_cast<const uint4*>(Dc + j);
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t lo = (j + 2 * e < s1) ? (uint32_t)(fromg ? __ldcg(Dc + j + 2 * e) : Dc[j + 2 * e]) : 0xffffu;
      const uint32_t hi = (j + 2 * e + 1 < s1) ? (uint32_t)(fromg ? __ldcg(Dc + j + 2 * e + 1) : Dc[j + 2 * e + 1])
                                               : 0xffffu;
      v[e] = lo | (hi << 16);
    }
  }
  ltm = 0;
  tim = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int dv = (int)((v[e >> 1] >> (16 * (e & 1))) & 0xffffu);
    ltm |= (uint32_t)(dv < thr) << e;
    tim |= (uint32_t)(dv == thr) << e;
  }
}

// Order-preserving compaction over the chunks ch[0..nch) at once: the warps
// are split evenly between the chunks; a lane owns 8 consecutive tokens, a
// warp a contiguous segment.  Token t of chunk c is selected iff D < thr, or
// D == thr and its tie rank within the chunk is < quota; its selection
// position is base + #selected before it in the chunk.  Positions in
// [P0, P1) are passed to emit(pos, token, D).  All threads must call.
template <typename Emit>
__device__ __forceinline__ void scan_chunks(const ChunkRef* ch, int nch, int thr, int P0, int P1, int* wcnt,
                                            Emit emit) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int c0 = 0; c0 < nch; c0 += DEC_WARPS) {
    const int n_here = min(DEC_WARPS, nch - c0);
    const int wpc = DEC_WARPS / n_here;                 // warps per chunk
    const int ci = warp / wpc, sub = warp % wpc;
    const bool active = ci < n_here;
    ChunkRef c = {};
    if (active) c = ch[c0 + ci];
    const int seg = ((c.L + wpc - 1) / wpc + 255) & ~255;
    const int s0 = active ? min(c.L, sub * seg) : 0, s1 = active ? min(c.L, s0 + seg) : 0;
    int lt_w = 0, ti_w = 0;
    for (int j0 = s0; j0 < s1; j0 += 256) {
      uint32_t ltm = 0, tim = 0;
      if (j0 + 8 * lane < s1) d_masks(c.D, c.fromg, j0 + 8 * lane, s1, thr, ltm, tim);
      lt_w += __popc(ltm);
      ti_w += __popc(tim);
    }
    lt_w = warp_sum_i(lt_w);
    ti_w = warp_sum_i(ti_w);
    __syncthreads();                                   // wcnt reuse guard
    if (lane == 0) { wcnt[2 * warp] = lt_w; wcnt[2 * warp + 1] = ti_w; }
    __syncthreads();
    if (active) {
      int lt_b = 0, ti_b = 0;
      for (int w = ci * wpc; w < warp; ++w) { lt_b += wcnt[2 * w]; ti_b += wcnt[2 * w + 1]; }
      const int q = c.quota, base = c.base;
      const int seg_first = base + lt_b + min(ti_b, q);
      const int seg_last = base + lt_b + lt_w + min(ti_b + ti_w, q);   // exclusive
      if (seg_last > P0 && seg_first < P1) {
        for (int j0 = s0; j0 < s1; j0 += 256) {
          const int j = j0 + 8 * lane;
          uint32_t ltm = 0, tim = 0;
          if (j < s1) d_masks(c.D, c.fromg, j, s1, thr, ltm, tim);
          const int mine = __popc(ltm) | (__popc(tim) << 16);
          int incl = mine;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          const int excl = incl - mine;
          const int tot = __shfl_sync(0xffffffffu, incl, 31);
          const int ltl = lt_b + (excl & 0xffff), til = ti_b + (excl >> 16);
          uint32_t any = ltm | tim;
          while (any) {
            const int e = __ffs(any) - 1;
            any &= any - 1;
            const uint32_t below = (1u << e) - 1u;
            const int tr = til + __popc(tim & below);
            if (((ltm >> e) & 1u) || tr < q) {
              const int pos = base + ltl + __popc(ltm & below) + min(tr, q);
              if (pos >= P0 && pos < P1) {
                const int dv = c.fromg ? (int)__ldcg(c.D + j + e) : (int)c.D[j + e];
                emit(pos, c.tok0 + j + e, dv);
              }
            }
          }
          lt_b += tot & 0xffff;
          ti_b += tot >> 16;
        }
      }
    }
  }
}

template <typename T, int W, int GT, int D_HEAD>
__global__ void __launch_bounds__(DEC_THREADS, 1) hata_decode_kernel(const __grid_constant__ DecodeParams p) {
  constexpr int J = planes_for_group(GT);
  constexpr int STAGE_TOK = DEC_STAGE_BYTES / (W * 4);
  constexpr int EB = sizeof(T);
  constexpr int NSL = AttnState<GT, D_HEAD>::NSL;
  extern __shared__ __align__(1024) uint8_t smem[];
  HATA_TRACE(31);
  if (p.dbg & 4) return;                                           // diagnostics: launch cost only

  const int M = p.M;
  const int NST = p.stages;
  const int r = blockIdx.x;
  const int u = blockIdx.y;
  const int b = u / p.Hkv, g = u % p.Hkv;
  const int G = p.G;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const DecodeSmem L = decode_smem_layout(p, GT, EB);
  const int QS = dec_qstride(D_HEAD);

  uint8_t* ring = smem + L.ring;
  T* Ws = reinterpret_cast<T*>(smem + L.W);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);  // [NST] ring, [NST] W, [NST+1] exchange, [NST+2] partials
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem + L.hist);
  uint16_t* Dglob = p.ws_D ? p.ws_D + ((int64_t)u * M + r) * p.chunk : nullptr;
  uint16_t* Dloc = p.d_smem ? reinterpret_cast<uint16_t*>(smem + L.D) : Dglob;
  float* qf = reinterpret_cast<float*>(smem + L.qf);
  uint32_t* qw = reinterpret_cast<uint32_t*>(smem + L.qw);
  uint32_t* planes = reinterpret_cast<uint32_t*>(smem + L.planes);   // [2][4][8]
  int32_t* rows = p.ws_rows ? p.ws_rows + ((int64_t)u * M + r) * p.R_cap : reinterpret_cast<int32_t*>(smem + L.rows);
  int32_t* red = reinterpret_cast<int32_t*>(smem + L.red);
  int32_t* misc = reinterpret_cast<int32_t*>(smem + L.misc);
  float* fmisc = reinterpret_cast<float*>(misc);

  // Rank chunks [rr*per, (rr+1)*per) are fixed by the host from n_max, so the
  // streams start before the device-side length n[b] has arrived.
  const int per = p.chunk;
  const int64_t t0 = (int64_t)r * per;
  const int Lcopy = (int)max((int64_t)0, min((int64_t)per, p.n_max - t0));   // rows streamed
  const int nstages = (Lcopy + STAGE_TOK - 1) / STAGE_TOK;
  const bool recycle = nstages > NST;                              // ring smaller than the chunk
  const uint32_t* cbase = p.codes + (int64_t)b * p.c_sb + (int64_t)g * p.c_sh;
  const T* qg = reinterpret_cast<const T*>(p.q) + ((int64_t)b * p.Hq + (int64_t)g * G) * D_HEAD;
  const bool append = p.k_new != nullptr;
  T* qraw = reinterpret_cast<T*>(smem + L.qraw);                    // [G (+1 key)][d] as stored

  // ---- phase 0: start every stream: the code chunk by a few large bulk copies
  // (TMA), W_g / q / the new key by coalesced 16-byte loads of all threads
  auto issue_stage = [&](int s) {
    const int slot = s % NST;
    const int ntok = min(STAGE_TOK, Lcopy - s * STAGE_TOK);
    const uint32_t bytes = (uint32_t)(ntok * W * 4) & ~15u;
    mbar_arrive_expect_tx(&bars[slot], bytes);
    if (bytes) bulk_g2s(ring + slot * DEC_STAGE_BYTES, cbase + (t0 + (int64_t)s * STAGE_TOK) * W, bytes, &bars[slot]);
  };
  const int64_t n = p.n[b];                                         // requested before the streams
  const int wrow = p.rbits * EB;                                    // bytes of one W row
  const int WROWB = dec_wrow_stride(p.rbits, EB);                   // padded smem row (bank spread)
  {
    constexpr int MAXC = 8;                                          // 16-byte chunks per thread (<= 64 KB)
    const uint4* wsrc = reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(p.Wh) + (int64_t)g * p.d * p.rbits);
    const int cpr = wrow / 16, nwc = D_HEAD * cpr;                 // chunks per row / in W_g
    uint4 v[MAXC];
    // W_g beyond MAXC chunks per thread (fp32 with rbits = 256): earlier batches
    for (int base = 0; base + MAXC * DEC_THREADS < nwc; base += MAXC * DEC_THREADS) {
#pragma unroll
      for (int c = 0; c < MAXC; ++c) v[c] = __ldg(wsrc + base + tid + c * DEC_THREADS);
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        const int i = base + tid + c * DEC_THREADS;
        *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(Ws) + (i / cpr) * WROWB + (i % cpr) * 16) = v[c];
      }
    }
    const int wlast = (nwc - 1) / (MAXC * DEC_THREADS) * (MAXC * DEC_THREADS);   // last batch
#pragma unroll
    for (int c = 0; c < MAXC; ++c)
      if (wlast + tid + c * DEC_THREADS < nwc) v[c] = __ldg(wsrc + wlast + tid + c * DEC_THREADS);
    const int nq = G * D_HEAD * EB / 16, nk = append ? D_HEAD * EB / 16 : 0;
    uint4 vq = make_uint4(0, 0, 0, 0);
    const uint4* qsrc = reinterpret_cast<const uint4*>(qg);
    const uint4* ksrc = reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(p.k_new) + (int64_t)u * D_HEAD);
    if (tid < nq) vq = __ldg(qsrc + tid);
    else if (tid < nq + nk) vq = __ldg(ksrc + (tid - nq));
    // the small loads above are in flight ahead of the 128 KB code stream
    if (tid == 0) {
      // [0, NST) code ring, NST: unused, NST+1: exchange + D staging, NST+2: partials,
      // NST+3: attention gather batches
      for (int s = 0; s < NST + 4; ++s) mbar_init(&bars[s], 1);
      fence_mbar_init();
      for (int s = 0; s < NST && s < nstages; ++s) issue_stage(s);
    }
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const int i = wlast + tid + c * DEC_THREADS;
      if (i < nwc) *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(Ws) + (i / cpr) * WROWB + (i % cpr) * 16) = v[c];
    }
    if (tid < nq + nk) reinterpret_cast<uint4*>(qraw)[tid] = vq;
  }
  for (int i = tid; i < p.nbins; i += DEC_THREADS) hist[i] = 0;
  const int kp = (int)(n < (int64_t)p.k ? n : (int64_t)p.k);      // k' = min(k, n)  (R10)
  auto chunk_len = [&](int rr) -> int {                            // valid tokens of rank rr
    const int64_t a = (int64_t)rr * per, z = min((int64_t)n, a + per);
    return z > a ? (int)(z - a) : 0;
  };
  const int Lr = chunk_len(r);

  HATA_TRACE(0);
  // ---- phase 1: Encode & Cache update (Alg. 3 lines 2-9; fused as
  // in §4): hash the G query heads of the group and, when this launch
  // also appends the new token (k_new != null), its key -- one projection pass
  // with the key as row G.  The rank owning row pos = n-1 writes K/V/code rows.
  const int64_t pos = n - 1;
  const bool owner = append && n >= 1 && pos >= t0 && pos < t0 + Lr;
  const int NV = G + (owner ? 1 : 0);                                // projected vectors
  __syncthreads();                                                  // W_g, q, k_new in smem
  HATA_TRACE(9);
  for (int i = tid; i < NV * D_HEAD; i += DEC_THREADS) qf[(i / D_HEAD) * QS + i % D_HEAD] = Elem<T>::to_f(qraw[i]);
  if (owner) {
    const T* vn = reinterpret_cast<const T*>(p.v_new) + (int64_t)u * D_HEAD;
    T* Kd = const_cast<T*>(reinterpret_cast<const T*>(p.K)) + (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh + pos * p.kv_st;
    T* Vd = const_cast<T*>(reinterpret_cast<const T*>(p.V)) + (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh + pos * p.kv_st;
    for (int i = tid; i < D_HEAD; i += DEC_THREADS) {
      Kd[i] = qraw[G * D_HEAD + i];                                    // Alg. 3 line 3
      Vd[i] = vn[i];                                                   // Alg. 3 line 4
    }
  }
  __syncthreads();
  HATA_TRACE(8);
  if constexpr (EB == 2) {
    // bf16: the projection X[NV x d] . W_g[d x rbits] on the tensor cores
    // (mma.sync m16n8k16, exact bf16 products, fp32 accumulation; R13).
    // Warp = one 8-bit column tile of the code; Sign + BitPack (Alg. 2 lines
    // 5-7) straight from the accumulator fragment via ballots.
    const int gid = lane >> 2, tig = lane & 3;
    uint8_t* qbytes = reinterpret_cast<uint8_t*>(qw);               // [GT+1][W*4] code bytes
    for (int nt = warp; nt < p.rbits / 8; nt += DEC_WARPS) {
      float c[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int k0 = 0; k0 < D_HEAD; k0 += 16) {
        uint32_t a[4];
        const float* x0 = qf + gid * QS + k0 + 2 * tig;
        const float* x1 = qf + (gid + 8) * QS + k0 + 2 * tig;
        const float2 z = make_float2(0.f, 0.f);
        const float2 f0 = gid < NV ? *reinterpret_cast<const float2*>(x0) : z;
        const float2 f1 = gid + 8 < NV ? *reinterpret_cast<const float2*>(x1) : z;
        const float2 f2 = gid < NV ? *reinterpret_cast<const float2*>(x0 + 8) : z;
        const float2 f3 = gid + 8 < NV ? *reinterpret_cast<const float2*>(x1 + 8) : z;
        a[0] = pack_bf16x2(f0.x, f0.y);                             // exact: q, k are bf16
        a[1] = pack_bf16x2(f1.x, f1.y);
        a[2] = pack_bf16x2(f2.x, f2.y);
        a[3] = pack_bf16x2(f3.x, f3.y);
        uint32_t b0, b1;
        ldsm_x2_trans(b0, b1, reinterpret_cast<const uint8_t*>(Ws) + (k0 + (lane & 15)) * WROWB + nt * 16);
        mma_bf16_16816(c, a, b0, b1);
      }
      const uint32_t m0 = __ballot_sync(0xffffffffu, c[0] >= 0.f), m1 = __ballot_sync(0xffffffffu, c[1] >= 0.f);
      const uint32_t m2 = __ballot_sync(0xffffffffu, c[2] >= 0.f), m3 = __ballot_sync(0xffffffffu, c[3] >= 0.f);
      if (tig == 0) {
        uint32_t lo = 0, hi = 0;                                    // bits nt*8 .. nt*8+7, LSB-first (R7)
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          lo |= ((m0 >> (gid * 4 + t)) & 1u) << (2 * t) | ((m1 >> (gid * 4 + t)) & 1u) << (2 * t + 1);
          hi |= ((m2 >> (gid * 4 + t)) & 1u) << (2 * t) | ((m3 >> (gid * 4 + t)) & 1u) << (2 * t + 1);
        }
        if (gid < NV) qbytes[gid * W * 4 + nt] = (uint8_t)lo;
        if (gid + 8 < NV) qbytes[(gid + 8) * W * 4 + nt] = (uint8_t)hi;
      }
    }
  } else {
    // fp32: thread = (bit, j-slice), all vectors at once (fp32 FMA; slices
    // summed in fixed order), then Sign + BitPack by ballots
    float* qpart = reinterpret_cast<float*>(smem + L.qp);           // [nparts][GT+1][rbits]
    const int nparts = DEC_THREADS / p.rbits;
    const int bit = tid % p.rbits, part = tid / p.rbits;           // part is warp-uniform
    const int jlen = D_HEAD / nparts;
    const int wstride = WROWB / EB;
    float acc[GT + 1];
#pragma unroll
    for (int h = 0; h <= GT; ++h) acc[h] = 0.f;
    const T* wc = Ws + bit;
    for (int j0 = part * jlen; j0 < (part + 1) * jlen; j0 += 4) {
      float wv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) wv[e] = Elem<T>::to_f(wc[(j0 + e) * wstride]);
#pragma unroll
      for (int h = 0; h <= GT; ++h) {
        if (h < NV) {
          const float4 qv = *reinterpret_cast<const float4*>(qf + h * QS + j0);
          acc[h] = fmaf(qv.x, wv[0], acc[h]);
          acc[h] = fmaf(qv.y, wv[1], acc[h]);
          acc[h] = fmaf(qv.z, wv[2], acc[h]);
          acc[h] = fmaf(qv.w, wv[3], acc[h]);
        }
      }
    }
#pragma unroll
    for (int h = 0; h <= GT; ++h)
      if (h < NV) qpart[(part * (GT + 1) + h) * p.rbits + bit] = acc[h];
    __syncthreads();
    for (int o = tid; o < NV * p.rbits; o += DEC_THREADS) {
      const int h = o / p.rbits, bb = o % p.rbits;
      float sum = 0.f;
      for (int pp = 0; pp < nparts; ++pp) sum += qpart[(pp * (GT + 1) + h) * p.rbits + bb];
      const uint32_t word = __ballot_sync(0xffffffffu, sum >= 0.f);
      if (lane == 0) qw[h * W + bb / 32] = word;
    }
  }
  __syncthreads();
  // publish the query codes (optional output) and the new key's code (Alg. 3 line 9)
  for (int i = tid; i < NV * W; i += DEC_THREADS) {
    const int h = i / W, w = i % W;
    const uint32_t word = qw[i];
    if (h < G && p.out_qcodes && r == 0) p.out_qcodes[((int64_t)b * p.Hq + g * G + h) * W + w] = word;
    if (h == G) const_cast<uint32_t*>(p.codes)[(int64_t)b * p.c_sb + (int64_t)g * p.c_sh + pos * W + w] = word;
  }
  // bit planes of c_b = #{h: q_h bit b set} and of G - c_b (hata_score.cuh)
  if (warp < W) {
    int c = 0;
    for (int h = 0; h < G; ++h) c += (qw[h * W + warp] >> lane) & 1u;
    const int gc = G - c;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const uint32_t a = __ballot_sync(0xffffffffu, (c >> j) & 1);
      const uint32_t bb = __ballot_sync(0xffffffffu, (gc >> j) & 1);
      if (lane == 0) { planes[j * 8 + warp] = a; planes[32 + j * 8 + warp] = bb; }
    }
  }
  __syncthreads();
  uint32_t A[J][W], Bp[J][W];
#pragma unroll
  for (int j = 0; j < J; ++j)
#pragma unroll
    for (int w = 0; w < W; ++w) { A[j][w] = planes[j * 8 + w]; Bp[j][w] = planes[32 + j * 8 + w]; }

  HATA_TRACE(1);
  // ---- phase 2: Hamming score + GQA sum (Alg. 3 lines 10-11) + histogram
  const bool mirror = (M > 1) && p.d_smem;          // D also needed by the other ranks
  auto smem_code = [&](const uint32_t* st, int j, uint32_t (&kc)[W]) {
    if constexpr (W == 4) {
      const uint4 v = reinterpret_cast<const uint4*>(st)[j];
      kc[0] = v.x; kc[1] = v.y; kc[2] = v.z; kc[3] = v.w;
    } else if constexpr (W == 8) {
      const uint4 v0 = reinterpret_cast<const uint4*>(st)[2 * j], v1 = reinterpret_cast<const uint4*>(st)[2 * j + 1];
      kc[0] = v0.x; kc[1] = v0.y; kc[2] = v0.z; kc[3] = v0.w; kc[4] = v1.x; kc[5] = v1.y; kc[6] = v1.z; kc[7] = v1.w;
    } else {
#pragma unroll
      for (int w = 0; w < W; ++w) kc[w] = st[j * W + w];
    }
  };
  int slot = 0;
  uint32_t parity = 0;
  for (int s = 0; s < nstages; ++s) {
    mbar_wait(&bars[slot], parity);
    if (s == 0) HATA_TRACE(10);
    if (s == nstages - 1) HATA_TRACE(13);
    const int base = s * STAGE_TOK;
    const int nval = min(STAGE_TOK, Lr - base);                     // valid tokens (< n), may be <= 0
    const int copied = (int)(((uint32_t)(min(STAGE_TOK, Lcopy - base) * W * 4) & ~15u) / (W * 4));
    const int npairs = max(0, min(nval, copied)) / 2;
    const uint32_t* st = reinterpret_cast<const uint32_t*>(ring + slot * DEC_STAGE_BYTES);
    uint32_t* dst = reinterpret_cast<uint32_t*>(Dloc + base);
    uint32_t* dst2 = mirror ? reinterpret_cast<uint32_t*>(Dglob + base) : nullptr;
    // two tokens per thread per iteration -> one 32-bit store of a u16 pair
    for (int j2 = tid; j2 < npairs; j2 += DEC_THREADS) {
      uint32_t k0[W], k1[W];
      smem_code(st, 2 * j2, k0);
      smem_code(st, 2 * j2 + 1, k1);
      const uint32_t d0 = group_distance<W, J>(k0, A, Bp);
      const uint32_t d1 = group_distance<W, J>(k1, A, Bp);
      atomicAdd(&hist[d0], 1u);
      atomicAdd(&hist[d1], 1u);
      const uint32_t packed = d0 | (d1 << 16);
      dst[j2] = packed;
      if (mirror) dst2[j2] = packed;
    }
    // leftovers: an odd last token, or tokens past the 16-byte-rounded copy
    const int rest = nval - 2 * npairs;
    if (tid < rest) {
      const int j = 2 * npairs + tid;
      uint32_t kc[W];
      if (j < copied) {
        smem_code(st, j, kc);
      } else {
        const uint32_t* gp = cbase + (t0 + base + j) * W;
#pragma unroll
        for (int w = 0; w < W; ++w) kc[w] = __ldg(gp + w);
      }
      const uint32_t dv = group_distance<W, J>(kc, A, Bp);
      atomicAdd(&hist[dv], 1u);
      Dloc[base + j] = (uint16_t)dv;
      if (mirror) Dglob[base + j] = (uint16_t)dv;
    }
    if (recycle) {                                                  // refill the slot just consumed
      __syncthreads();
      if (tid == 0 && s + NST < nstages) issue_stage(s + NST);
    }
    if (++slot == NST) { slot = 0; parity ^= 1u; }
  }
  __syncthreads();                                                  // every D / histogram update done
  if (owner && tid == 0) {
    // the streamed row pos held the stale code: re-score the appended key
    uint32_t kc[W];
#pragma unroll
    for (int w = 0; w < W; ++w) kc[w] = qw[G * W + w];
    const int jl = (int)(pos - t0);
    const uint32_t Dn = group_distance<W, J>(kc, A, Bp);
    const uint32_t Do = Dloc[jl];
    hist[Do] -= 1u;
    hist[Dn] += 1u;
    Dloc[jl] = (uint16_t)Dn;
    if (mirror) Dglob[jl] = (uint16_t)Dn;
  }
  __syncthreads();

  // ---- phase 3: exact top-k' (Alg. 3 lines 12-13) by counting select.
  // thr = D of the k'-th best token; every D < thr is selected; ties at thr
  // are taken lowest index first (R8) through per-rank quotas in rank (=
  // token) order.  The ranks of a unit exchange histograms exactly once.
  const int hs = dec_hist_stride(p.nbins);                          // 16-byte rows
  int32_t* hm = reinterpret_cast<int32_t*>(smem + L.hm);           // [M][hs]  (ring+W area)
  unsigned* sync = (M > 1) ? p.ws_sync + 2 * u : nullptr;
  HATA_TRACE(2);
  if (M > 1) {
    int32_t* gh = p.ws_hist + ((int64_t)u * M + r) * hs;
    for (int i = tid; i < p.nbins; i += DEC_THREADS) gh[i] = (int32_t)hist[i];
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      atomicAdd(sync, 1u);
    }
    // While the other ranks finish scoring: warm L2 with the K/V rows this
    // rank will most likely select (its own tokens below a local estimate of
    // the threshold), so the gather after the selection hits L2.  A pure
    // prefetch: the selection itself is decided exactly after the exchange.
    if (!p.cand_mode && !(p.dbg & 2)) {
      const int want = (int)(((int64_t)kp * Lr + n - 1) / (n > 0 ? n : 1)) * 9 / 8 + 4;
      int mysum = 0, tb[5];
      const int BPT = (p.nbins + DEC_THREADS - 1) / DEC_THREADS, i0 = tid * BPT;
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        tb[q] = (q < BPT && i0 + q < p.nbins) ? (int)hist[i0 + q] : 0;
        mysum += tb[q];
      }
      int total;
      int cum = block_excl_scan(mysum, misc + 16, total);
      if (tid == 0) misc[4] = p.nbins;
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        if (cum < want && cum + tb[q] >= want) misc[4] = i0 + q;
        cum += tb[q];
      }
      __syncthreads();
      const int test = misc[4];                                     // prefetch tokens with D <= test
      const __nv_bfloat16* Kb = reinterpret_cast<const __nv_bfloat16*>(p.K) + (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh;
      const __nv_bfloat16* Vb = reinterpret_cast<const __nv_bfloat16*>(p.V) + (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh;
      for (int j = tid * 8; j < Lr; j += DEC_THREADS * 8) {
        uint32_t ltm, tim;
        d_masks(Dloc, !p.d_smem, j, Lr, test + 1, ltm, tim);
        while (ltm) {
          const int e = __ffs(ltm) - 1;
          ltm &= ltm - 1;
          const int64_t t = t0 + j + e;
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(Kb + t * p.kv_st), "r"(D_HEAD * EB) : "memory");
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(Vb + t * p.kv_st), "r"(D_HEAD * EB) : "memory");
        }
      }
    }
    if (tid == 0) {
      while (ld_acquire_gpu(sync) < (unsigned)M) {
      }
      // other ranks' generic-proxy writes -> this thread's async-proxy (bulk copy) reads
      asm volatile("fence.proxy.async.global;" ::: "memory");
      const uint32_t bytes = (uint32_t)(M * hs * 4);
      mbar_arrive_expect_tx(&bars[NST + 1], bytes);
      bulk_g2s(hm, p.ws_hist + (int64_t)u * M * hs, bytes, &bars[NST + 1]);
    }
    mbar_wait(&bars[NST + 1], 0);
  } else {
    for (int i = tid; i < p.nbins; i += DEC_THREADS) hm[i] = (int32_t)hist[i];
    __syncthreads();
  }
  HATA_TRACE(3);
  // (a) per-bin totals over the ranks + block scan -> thr, #below
  {
    constexpr int BPT_MAX = 5;                                       // nbins <= 2560
    const int BPT = (p.nbins + DEC_THREADS - 1) / DEC_THREADS;
    const int i0 = tid * BPT;
    int tb[BPT_MAX];
    int mysum = 0;
#pragma unroll
    for (int q = 0; q < BPT_MAX; ++q) {
      tb[q] = 0;
      const int i = i0 + q;
      if (q < BPT && i < p.nbins) {
        int s0 = 0, s1 = 0, s2 = 0, s3 = 0, rr = 0;
        for (; rr + 4 <= M; rr += 4) {
          s0 += hm[rr * hs + i]; s1 += hm[(rr + 1) * hs + i]; s2 += hm[(rr + 2) * hs + i]; s3 += hm[(rr + 3) * hs + i];
        }
        for (; rr < M; ++rr) s0 += hm[rr * hs + i];
        tb[q] = s0 + s1 + s2 + s3;
      }
      mysum += tb[q];
    }
    int total;
    int cum = block_excl_scan(mysum, misc + 16, total);
    if (tid == 0 && kp <= 0) { misc[0] = -1; misc[1] = 0; }
#pragma unroll
    for (int q = 0; q < BPT_MAX; ++q) {
      if (q < BPT && i0 + q < p.nbins && kp > 0 && cum < kp && cum + tb[q] >= kp) {
        misc[0] = i0 + q;          // thr
        misc[1] = kp - cum;        // need: ties to take at thr
      }
      cum += tb[q];
    }
  }
  __syncthreads();
  HATA_TRACE(11);
  const int thr = misc[0];
  const int need = misc[1];
  // (b) per-rank #(D < thr) and #(D == thr): warp per rank
  int32_t* rb_below = red;                       // [M]
  int32_t* rb_ties = red + DEC_MAX_RANKS;        // [M]
  int32_t* rb_off = red + 2 * DEC_MAX_RANKS;     // [M]
  int32_t* rb_quota = red + 3 * DEC_MAX_RANKS;   // [M]
  for (int rr = warp; rr < M; rr += DEC_WARPS) {
    int s0 = 0, s1 = 0, s2 = 0, s3 = 0, i = lane;
    for (; i + 96 < thr; i += 128) {
      s0 += hm[rr * hs + i]; s1 += hm[rr * hs + i + 32]; s2 += hm[rr * hs + i + 64]; s3 += hm[rr * hs + i + 96];
    }
    for (; i < thr; i += 32) s0 += hm[rr * hs + i];
    const int s = warp_sum_i(s0 + s1 + s2 + s3);
    if (lane == 0) { rb_below[rr] = s; rb_ties[rr] = thr >= 0 ? hm[rr * hs + thr] : 0; }
  }
  __syncthreads();
  // (c) quotas, selection offsets, and staging of the D arrays this rank needs
  const int R = (kp + M - 1) / M;                                   // equal share of the selection
  const int P0 = min(kp, r * R), P1 = min(kp, P0 + R);
  ChunkRef* chref = reinterpret_cast<ChunkRef*>(smem + L.chref);   // [DEC_MAX_RANKS]
  if (warp == 0) {
    const int bl = lane < M ? rb_below[lane] : 0, ti = lane < M ? rb_ties[lane] : 0;
    int incl = ti;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int quota = max(0, min(need - (incl - ti), ti));
    const int sel = bl + quota;
    int inc2 = sel;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc2, o);
      if (lane >= o) inc2 += v;
    }
    const int off = inc2 - sel;
    if (lane < M) { rb_quota[lane] = quota; rb_off[lane] = off; }
    // chunks whose selections overlap [P0, P1): a contiguous run of ranks
    const bool ov = lane < M && P1 > P0 && sel > 0 && off < P1 && off + sel > P0;
    const uint32_t ovm = __ballot_sync(0xffffffffu, ov);
    const bool own = lane == r && p.d_smem;
    const int Lc = lane < M ? chunk_len(lane) : 0;
    uint32_t bytes = (ov && !own) ? (uint32_t)((Lc * 2 + 15) & ~15) : 0u;
    // smem slots after the histograms, in rank order
    uint32_t slot = (bytes + 127) & ~127u, sx = slot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, sx, o);
      if (lane >= o) sx += v;
    }
    const uint32_t soff = (uint32_t)((M * hs * 4 + 127) & ~127) + sx - slot;
    if (soff + bytes > (uint32_t)L.sc_limit) bytes = 0;            // does not fit: scan it in L2
    const uint32_t tx = (uint32_t)warp_sum_i((int)bytes);
    if (ov) {
      const int k = __popc(ovm & ((1u << lane) - 1u));
      ChunkRef c;
      c.L = Lc;
      c.quota = quota;
      c.base = off;
      c.tok0 = lane * per;
      c.fromg = (!own && !bytes) ? 1 : 0;
      c.D = own ? Dloc : (bytes ? reinterpret_cast<const uint16_t*>(smem + soff)
                                : p.ws_D + ((int64_t)u * M + lane) * p.chunk);
      chref[k] = c;
    }
    if (lane == 0) { misc[2] = __popc(ovm); misc[3] = tx ? 1 : 0; }
    if (tx) {
      if (lane == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");     // D written by generic stores
        mbar_arrive_expect_tx(&bars[NST + 1], tx);
      }
      __syncwarp();
      if (bytes) bulk_g2s(smem + soff, p.ws_D + ((int64_t)u * M + lane) * p.chunk, bytes, &bars[NST + 1]);
    }
  }
  __syncthreads();
  HATA_TRACE(12);
  const int nch = misc[2];
  if (misc[3]) mbar_wait(&bars[NST + 1], M > 1 ? 1 : 0);
  HATA_TRACE(4);
  int32_t* oidx = p.out_idx ? p.out_idx + (int64_t)u * p.k : nullptr;
  int32_t* osc = p.out_score ? p.out_score + (int64_t)u * p.k : nullptr;
  int32_t* ocd = p.cand_D ? p.cand_D + (int64_t)u * p.k : nullptr;
  const int Gr = G * p.rbits;
  scan_chunks(chref, nch, thr, P0, P1, misc + 32, [&](int pos, int tok, int Dv) {
    rows[pos - P0] = tok;
    if (oidx) oidx[pos] = (int32_t)(tok + p.token_offset);
    if (osc) osc[pos] = Gr - 2 * Dv;                               // S = G*rbits - 2D
    if (ocd) ocd[pos] = Dv;
  });
  if (r == 0) {
    for (int i = kp + tid; i < p.k; i += DEC_THREADS) {
      if (oidx) oidx[i] = -1;
      if (osc) osc[i] = 0;
      if (ocd) ocd[i] = 0x7fffffff;
    }
  }
  __syncthreads();

  HATA_TRACE(5);
  // ---- phase 4: gather + softmax attention over this rank's rows (Alg. 3 lines 14-17)
  float* m_s = fmisc + 80;
  float* l_s = fmisc + 88;
  float* corr_s = fmisc + 96;
  AttnState<GT, D_HEAD> st;
  if (!p.cand_mode) {
    const T* Kb = reinterpret_cast<const T*>(p.K) + (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh;
    const T* Vb = reinterpret_cast<const T*>(p.V) + (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh;
    if constexpr (EB == 2) {
      attend_rows_mma<GT, D_HEAD>(rows, P1 - P0, Kb, Vb, p.kv_st, qf, G, p.scale, smem + L.kv, p.rows_cap, L.rb,
                                  m_s, l_s, st, &bars[NST + 3], p.trace);
    } else {
      float* sc = reinterpret_cast<float*>(smem + L.sc);
      attend_rows<T, GT, D_HEAD>(rows, P1 - P0, Kb, Vb, p.kv_st, qf, G, p.scale, smem + L.kv, sc, p.rows_cap, L.rb,
                                 m_s, l_s, corr_s, st);
    }
  }
  HATA_TRACE(6);

  // ---- phase 5: merge the M rank partials in rank order (flash-decoding combine)
  const int64_t orow = (int64_t)b * p.Hq + (int64_t)g * G;      // first output row of the group
  auto store_out = [&](int h, int e, float v) {
    const int64_t oi = (orow + h) * D_HEAD + e;
    if (p.out_bf16) reinterpret_cast<__nv_bfloat16*>(p.out)[oi] = __float2bfloat16_rn(v);
    else reinterpret_cast<float*>(p.out)[oi] = v;
  };
  if (M == 1) {
    if (!p.cand_mode) {
#pragma unroll
      for (int s = 0; s < NSL; ++s) {
        const int sl = tid + s * DEC_THREADS;
        const int h = sl / (D_HEAD / 2), e2 = sl % (D_HEAD / 2);
        if (h < G) {
          const float l = l_s[h];
          store_out(h, 2 * e2, l > 0.f ? st.acc[s][0] / l : 0.f);
          store_out(h, 2 * e2 + 1, l > 0.f ? st.acc[s][1] / l : 0.f);
        }
      }
    }
    HATA_TRACE(7);
    return;
  }
  const int PS = D_HEAD + 2;
  const int PB = dec_part_stride(GT, D_HEAD);
  float* mypart = p.ws_part + ((int64_t)u * M + r) * PB;
  if (!p.cand_mode) {
#pragma unroll
    for (int s = 0; s < NSL; ++s) {
      const int sl = tid + s * DEC_THREADS;
      const int h = sl / (D_HEAD / 2), e2 = sl % (D_HEAD / 2);
      if (h < G) { mypart[h * PS + 2 + 2 * e2] = st.acc[s][0]; mypart[h * PS + 3 + 2 * e2] = st.acc[s][1]; }
    }
    if (tid < G) { mypart[tid * PS] = m_s[tid]; mypart[tid * PS + 1] = l_s[tid]; }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(sync + 1, 1u);
    misc[2] = (prev == (unsigned)(M - 1));
  }
  __syncthreads();
  HATA_TRACE(15);
  if (!misc[2]) return;
  // last rank: every partial is visible (writer fence + counter); pull them
  // into smem with one bulk copy, then merge in rank order
  if (!p.cand_mode) {
    float* sp = reinterpret_cast<float*>(smem);                      // ring+W area is free
    float* wgt = reinterpret_cast<float*>(smem + L.hm + ((M * PB * 4 + 127) & ~127));   // [M][GT] weights
    if (tid == 0) {
      __threadfence();
      HATA_TRACE(24);
      asm volatile("fence.proxy.async.global;" ::: "memory");
      const uint32_t bytes = (uint32_t)(M * PB * 4);
      mbar_arrive_expect_tx(&bars[NST + 2], bytes);
      bulk_g2s(sp, p.ws_part + (int64_t)u * M * PB, bytes, &bars[NST + 2]);
      HATA_TRACE(25);
    }
    mbar_wait(&bars[NST + 2], 0);
    HATA_TRACE(26);
    // per-head max, then per-(rank, head) weights e^{m_r - M_h}, then L_h
    if (tid < G) {
      float Mx = -INFINITY;
      for (int rr = 0; rr < M; ++rr) Mx = fmaxf(Mx, sp[rr * PB + tid * PS]);
      m_s[tid] = Mx;
    }
    __syncthreads();
    for (int t = tid; t < M * G; t += DEC_THREADS) {
      const int rr = t / G, h = t % G;
      const float mr = sp[rr * PB + h * PS];
      wgt[rr * GT + h] = (mr == -INFINITY) ? 0.f : expf(mr - m_s[h]);
    }
    __syncthreads();
    if (tid < G) {
      float Ls = 0.f;
      for (int rr = 0; rr < M; ++rr) Ls = fmaf(sp[rr * PB + tid * PS + 1], wgt[rr * GT + tid], Ls);
      l_s[tid] = Ls;
    }
    __syncthreads();
    for (int o = tid; o < G * D_HEAD; o += DEC_THREADS) {
      const int h = o / D_HEAD, e = o % D_HEAD;
      float a0 = 0.f, a1 = 0.f;
      int rr = 0;
      for (; rr + 2 <= M; rr += 2) {
        a0 = fmaf(sp[rr * PB + h * PS + 2 + e], wgt[rr * GT + h], a0);
        a1 = fmaf(sp[(rr + 1) * PB + h * PS + 2 + e], wgt[(rr + 1) * GT + h], a1);
      }
      if (rr < M) a0 = fmaf(sp[rr * PB + h * PS + 2 + e], wgt[rr * GT + h], a0);
      const float Ls = l_s[h];
      store_out(h, e, Ls > 0.f ? (a0 + a1) / Ls : 0.f);
    }
  }
  if (tid == 0) { sync[0] = 0u; sync[1] = 0u; }     // leave the workspace zeroed for the next launch
  HATA_TRACE(7);
}

}  // namespace hata
