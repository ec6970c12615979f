// Fused HATA decode kernel: q-hash -> Hamming score + GQA aggregate -> exact
// top-k (lowest index wins) -> gather + online-softmax attention -> split
// combine, in ONE launch.  One thread-block cluster of C CTAs per (b, KV head);
// every cross-CTA step goes through DSMEM + barrier.cluster (no global
// atomics, no grid sync).
//
// PAPER: Alg. 3 lines 6, 10-17; §4.
// Readings R1-R20 are listed in DESIGN.md.
#pragma once
#include "hata_common.cuh"
#include "hata_score.cuh"

namespace hata {

constexpr int DEC_THREADS = 256;
constexpr int DEC_WARPS = DEC_THREADS / 32;
constexpr int DEC_STAGE_BYTES = 16384;      // one bulk copy of codes
constexpr int DEC_STAGES = 4;               // ring depth (64 KB)
constexpr int DEC_RING_BYTES = DEC_STAGE_BYTES * DEC_STAGES;
constexpr int DEC_D_SMEM_MAX = 16384;       // tokens/CTA whose D (u16) lives in smem
constexpr int DEC_SEL_SMEM_MAX = 4096;      // selected rows/CTA held in smem
constexpr int DEC_CHUNK_ALIGN = 64;         // tokens

struct DecodeParams {
  const void* q;           // [B, Hq, d] contiguous
  const void* K;           // cache, element strides below, d contiguous
  const void* V;
  int64_t kv_sb, kv_sh, kv_st;
  const uint32_t* codes;   // [B, Hkv, cap, W] word strides, row stride == W
  int64_t c_sb, c_sh;
  const void* Wh;          // [Hkv, d, rbits] contiguous
  const int64_t* n;        // [B] tokens incl. appended one (device)
  int B, Hq, Hkv, G, d, rbits, k;
  float scale;
  void* out;               // [B, Hq, d]
  int out_bf16;
  int32_t* out_idx;        // [B, Hkv, k] or null
  int32_t* out_score;      // [B, Hkv, k] or null
  uint32_t* out_qcodes;    // [B, Hq, W] or null
  uint16_t* gD;            // global D workspace [B*Hkv*C*chunk] or null (smem)
  int32_t* gsel;           // global selected-list workspace [B*Hkv*C*rows_cap] or null (smem)
  int C;                   // cluster size (CTAs per (b, g))
  int chunk;               // tokens per CTA (capacity), multiple of DEC_CHUNK_ALIGN
  int nbins;               // G*rbits + 1
  int rows_cap;            // selected rows per CTA (capacity)
  // sequence-shard phase 1 (hata_shard_candidates): stop after the select and
  // emit (D, global index) candidates instead of attending.
  int cand_mode;
  int64_t token_offset;    // global index of local token 0
  int32_t* cand_D;         // [B, Hkv, k] or null
};

struct DecodeSmem {
  int ring, bars, hist, D, qf, qw, planes, sel, red, pub, part, misc, total;
};

// Shared-memory carve-up; identical on host and device.
__host__ __device__ inline DecodeSmem decode_smem_layout(const DecodeParams& p, int GT, int elem_bytes) {
  auto up = [](int x) { return (x + 127) & ~127; };
  DecodeSmem s;
  int off = 0;
  int wp = DEC_WARPS * GT * (p.d + 2) * 4;        // per-warp softmax partials (aliases ring)
  int ring = DEC_RING_BYTES > wp ? DEC_RING_BYTES : wp;
  (void)elem_bytes;
  s.ring = off; off += up(ring);
  s.bars = off; off += up(DEC_STAGES * 8 + 8);
  s.hist = off; off += up(p.nbins * 4);
  s.D = off; off += (p.gD ? 0 : up(p.chunk * 2));
  s.qf = off; off += up(GT * p.d * 4);
  s.qw = off; off += up(GT * (p.rbits / 32) * 4);
  s.planes = off; off += up(2 * 4 * 8 * 4);
  s.sel = off; off += (p.gsel ? 0 : up(p.rows_cap * 4));
  int sl = (p.nbins + p.C - 1) / p.C;
  s.red = off; off += up((sl + 1) * 4);
  s.pub = off; off += up(64 * 4);
  s.part = off; off += up(GT * (p.d + 2) * 4);
  s.misc = off; off += up(64 * 4);
  s.total = off;
  return s;
}

// Projection of one fp32 vector x[d] (smem) onto 32 consecutive hash bits
// [bit0, bit0+32) of W_g, returned as one packed word (lane i -> bit i).
// Alg. 2: Sign(MatMul) then BitPack, LSB-first; sign(0) -> 1.
template <typename T>
__device__ __forceinline__ uint32_t hash_word_warp(const float* __restrict__ x, const T* __restrict__ Wg, int d,
                                                   int rbits, int bit0, int lane) {
  float acc = 0.f;
  const T* col = Wg + bit0 + lane;
#pragma unroll 8
  for (int j = 0; j < d; ++j) acc = fmaf(x[j], Elem<T>::to_f(col[(int64_t)j * rbits]), acc);
  return __ballot_sync(0xffffffffu, acc >= 0.f);
}

// Gather + online softmax over `Rr` selected rows (indices in `rows`), all G
// heads of the group; result = this CTA's partial (m, l, acc[d]) per head in
// `part` ([GT][d+2]).  Alg. 3 lines 14-17 with the gather fused
// into the attention loop: rows are never materialised in HBM.
// `wp` is >= DEC_WARPS*GT*(d+2) floats of scratch.  All threads must call.
template <typename T, int GT, int D_HEAD>
__device__ __forceinline__ void attend_rows(const int32_t* rows, int Rr, const T* __restrict__ Kb,
                                            const T* __restrict__ Vb, int64_t kv_st, const float* qf, int G,
                                            float scale, float* wp, float* part) {
  constexpr int EPL = D_HEAD / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float qreg[GT][EPL];
#pragma unroll
  for (int h = 0; h < GT; ++h)
#pragma unroll
    for (int e = 0; e < EPL; ++e) qreg[h][e] = (h < G) ? qf[h * D_HEAD + lane * EPL + e] * scale : 0.f;
  float m_[GT], l_[GT], acc[GT][EPL];
#pragma unroll
  for (int h = 0; h < GT; ++h) {
    m_[h] = -INFINITY; l_[h] = 0.f;
#pragma unroll
    for (int e = 0; e < EPL; ++e) acc[h][e] = 0.f;
  }
  constexpr int U = 4;                                                // rows in flight per warp
  for (int i0 = warp * U; i0 < Rr; i0 += DEC_WARPS * U) {
    float kv[U][EPL], vv[U][EPL];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i0 + u < Rr) {
        const int64_t t = rows[i0 + u];
        load_row_slice<T, EPL>(Kb + t * kv_st + lane * EPL, kv[u]);
        load_row_slice<T, EPL>(Vb + t * kv_st + lane * EPL, vv[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i0 + u < Rr) {
#pragma unroll
        for (int h = 0; h < GT; ++h) {
          if (h < G) {
            float z = 0.f;
#pragma unroll
            for (int e = 0; e < EPL; ++e) z = fmaf(qreg[h][e], kv[u][e], z);
            z = warp_sum(z);
            const float mn = fmaxf(m_[h], z);
            const float a = expf(m_[h] - mn), pz = expf(z - mn);
            l_[h] = l_[h] * a + pz;
#pragma unroll
            for (int e = 0; e < EPL; ++e) acc[h][e] = fmaf(acc[h][e], a, pz * vv[u][e]);
            m_[h] = mn;
          }
        }
      }
    }
  }
  // merge the warps' partials in fixed warp order -> CTA partial (m, l, acc)
  const int stride_h = D_HEAD + 2;
#pragma unroll
  for (int h = 0; h < GT; ++h) {
    if (h < G) {
      float* dst = wp + (warp * GT + h) * stride_h;
      if (lane == 0) { dst[0] = m_[h]; dst[1] = l_[h]; }
#pragma unroll
      for (int e = 0; e < EPL; ++e) dst[2 + lane * EPL + e] = acc[h][e];
    }
  }
  __syncthreads();
  for (int o = tid; o < G * stride_h; o += DEC_THREADS) {
    const int h = o / stride_h, e = o % stride_h;
    float M = -INFINITY;
    for (int w = 0; w < DEC_WARPS; ++w) M = fmaxf(M, wp[(w * GT + h) * stride_h]);
    float v = 0.f;
    if (e == 0) v = M;
    else {
      for (int w = 0; w < DEC_WARPS; ++w) {
        const float mw = wp[(w * GT + h) * stride_h];
        const float sc = (mw == -INFINITY) ? 0.f : expf(mw - M);
        v = fmaf(wp[(w * GT + h) * stride_h + e], sc, v);
      }
    }
    part[h * stride_h + e] = v;
  }
}

// Flash-decoding merge of the C CTA partials of a cluster, in rank order:
// M = max m_c, L = sum l_c e^{m_c - M}, o = sum acc_c e^{m_c - M} / L.
// Writes normalised outputs to out[(row_base + h) * d + e] (fp32 or bf16), or,
// if `raw` is non-null, the merged partial (M, L, A) to raw[(row_base+h)*(d+2)].
// Caller brackets with cluster.sync().
template <int D_HEAD>
__device__ __forceinline__ void cluster_combine(cg::cluster_group& cluster, float* part, int C, int r, int G,
                                                int64_t row_base, void* out, int out_bf16, float* raw) {
  const int tid = threadIdx.x;
  const int stride_h = D_HEAD + 2;
  const int nout = G * stride_h;                                      // includes the (m, l) slots
  const int per_cta = (nout + C - 1) / C;
  const int o_lo = r * per_cta, o_hi = min(nout, o_lo + per_cta);
  const int segl = tid & 15;                                          // lane-in-segment = source rank
  for (int ob = o_lo; ob < o_hi; ob += DEC_THREADS / 16) {          // uniform trip count
    const int o = ob + (tid >> 4);
    const bool valid = o < o_hi;
    const int h = valid ? o / stride_h : 0, e = valid ? o % stride_h : 0;
    float mc = -INFINITY, lc = 0.f, vc = 0.f;
    if (valid && segl < C) {
      const float* rp = cluster.map_shared_rank(part, segl) + h * stride_h;
      mc = rp[0]; lc = rp[1]; vc = rp[e];
    }
    float M = mc;
#pragma unroll
    for (int s = 8; s > 0; s >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, s, 16));
    const float sc = (mc == -INFINITY) ? 0.f : expf(mc - M);
    float Ls = lc * sc, Vs = (e >= 1) ? vc * sc : 0.f;
#pragma unroll
    for (int s = 1; s < 16; s <<= 1) {
      Ls += __shfl_xor_sync(0xffffffffu, Ls, s, 16);
      Vs += __shfl_xor_sync(0xffffffffu, Vs, s, 16);
    }
    if (valid && segl == 0) {
      if (raw) {
        raw[(row_base + h) * stride_h + e] = (e == 0) ? M : Vs;
      } else if (e >= 2) {
        const float ov = (Ls > 0.f) ? Vs / Ls : 0.f;
        const int64_t oi = (row_base + h) * D_HEAD + (e - 2);
        if (out_bf16) reinterpret_cast<__nv_bfloat16*>(out)[oi] = __float2bfloat16_rn(ov);
        else reinterpret_cast<float*>(out)[oi] = ov;
      }
    }
  }
}

template <typename T, int W, int GT, int D_HEAD>
__global__ void __launch_bounds__(DEC_THREADS, 1) hata_decode_kernel(const __grid_constant__ DecodeParams p) {
  constexpr int J = planes_for_group(GT);
  constexpr int EPL = D_HEAD / 32;               // head elements per lane
  constexpr int STAGE_TOK = DEC_STAGE_BYTES / (W * 4);
  extern __shared__ __align__(1024) uint8_t smem[];

  cg::cluster_group cluster = cg::this_cluster();
  const int C = p.C;
  const int r = (int)cluster.block_rank();
  const int bg = blockIdx.y;
  const int b = bg / p.Hkv, g = bg % p.Hkv;
  const int G = p.G;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const DecodeSmem L = decode_smem_layout(p, GT, sizeof(T));

  uint8_t* ring = smem + L.ring;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem + L.hist);
  uint16_t* Dbuf = p.gD ? p.gD + ((int64_t)bg * C + r) * p.chunk : reinterpret_cast<uint16_t*>(smem + L.D);
  float* qf = reinterpret_cast<float*>(smem + L.qf);
  uint32_t* qw = reinterpret_cast<uint32_t*>(smem + L.qw);
  uint32_t* planes = reinterpret_cast<uint32_t*>(smem + L.planes);   // [2][4][8]
  int32_t* sel = p.gsel ? p.gsel + ((int64_t)bg * C + r) * p.rows_cap : reinterpret_cast<int32_t*>(smem + L.sel);
  uint32_t* red = reinterpret_cast<uint32_t*>(smem + L.red);
  int32_t* pub = reinterpret_cast<int32_t*>(smem + L.pub);
  float* part = reinterpret_cast<float*>(smem + L.part);              // [GT][d+2]: m, l, acc[d]
  int32_t* misc = reinterpret_cast<int32_t*>(smem + L.misc);

  const int64_t n = p.n[b];
  const int kp = (int)(n < (int64_t)p.k ? n : (int64_t)p.k);      // k' = min(k, n)  (R10)
  // this CTA's token chunk [t0, t1)
  int64_t per = ((n + C - 1) / C + DEC_CHUNK_ALIGN - 1) / DEC_CHUNK_ALIGN * DEC_CHUNK_ALIGN;
  if (per > p.chunk) per = p.chunk;
  const int64_t t0 = (int64_t)r * per;
  const int64_t t1 = (t0 + per < n) ? t0 + per : n;
  const int Lr = t1 > t0 ? (int)(t1 - t0) : 0;
  const int nstages = (Lr + STAGE_TOK - 1) / STAGE_TOK;
  const uint32_t* cbase = p.codes + (int64_t)b * p.c_sb + (int64_t)g * p.c_sh;

  // ---- phase 0: kick off the code stream (q-independent) before anything else
  if (tid == 0) {
    for (int s = 0; s < DEC_STAGES; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue_stage = [&](int s) {
    const int slot = s % DEC_STAGES;
    const int ntok = min(STAGE_TOK, Lr - s * STAGE_TOK);
    const uint32_t bytes = (uint32_t)(ntok * W * 4) & ~15u;
    if (bytes) {
      mbar_arrive_expect_tx(&bars[slot], bytes);
      bulk_g2s(ring + slot * DEC_STAGE_BYTES, cbase + (t0 + (int64_t)s * STAGE_TOK) * W, bytes, &bars[slot]);
    } else {
      mbar_arrive_expect_tx(&bars[slot], 0);
    }
  };
  if (tid == 0) {
    for (int s = 0; s < DEC_STAGES && s < nstages; ++s) issue_stage(s);
  }
  for (int i = tid; i < p.nbins; i += DEC_THREADS) hist[i] = 0;

  // ---- phase 1: q -> fp32 smem, hash the G query heads (Alg. 3 line 6)
  const T* qg = reinterpret_cast<const T*>(p.q) + ((int64_t)b * p.Hq + (int64_t)g * G) * p.d;
  for (int i = tid; i < G * p.d; i += DEC_THREADS) qf[i] = Elem<T>::to_f(qg[i]);
  __syncthreads();
  const T* Wg = reinterpret_cast<const T*>(p.Wh) + (int64_t)g * p.d * p.rbits;
  for (int wi = warp; wi < G * W; wi += DEC_WARPS) {
    const int h = wi / W, w = wi % W;
    uint32_t word = hash_word_warp<T>(qf + h * p.d, Wg, p.d, p.rbits, w * 32, lane);
    if (lane == 0) {
      qw[h * W + w] = word;
      if (p.out_qcodes && r == 0) p.out_qcodes[((int64_t)b * p.Hq + g * G + h) * W + w] = word;
    }
  }
  __syncthreads();
  // bit planes of c_b = #{h: q_h bit b set} and of G - c_b
  if (warp < W) {
    int c = 0;
    for (int h = 0; h < G; ++h) c += (qw[h * W + warp] >> lane) & 1u;
    const int gc = G - c;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      uint32_t a = __ballot_sync(0xffffffffu, (c >> j) & 1);
      uint32_t bb = __ballot_sync(0xffffffffu, (gc >> j) & 1);
      if (lane == 0) { planes[0 * 32 + j * 8 + warp] = a; planes[1 * 32 + j * 8 + warp] = bb; }
    }
  }
  __syncthreads();
  uint32_t A[J][W], Bp[J][W];
#pragma unroll
  for (int j = 0; j < J; ++j)
#pragma unroll
    for (int w = 0; w < W; ++w) { A[j][w] = planes[j * 8 + w]; Bp[j][w] = planes[32 + j * 8 + w]; }

  // ---- phase 2: Hamming score + GQA sum (Alg. 3 lines 10-11) + histogram
  for (int s = 0; s < nstages; ++s) {
    const int slot = s % DEC_STAGES;
    mbar_wait(&bars[slot], (s / DEC_STAGES) & 1);
    const int ntok = min(STAGE_TOK, Lr - s * STAGE_TOK);
    const int copied = (int)(((uint32_t)(ntok * W * 4) & ~15u) / (W * 4));
    const uint32_t* st = reinterpret_cast<const uint32_t*>(ring + slot * DEC_STAGE_BYTES);
    const int base = s * STAGE_TOK;
#pragma unroll 2
    for (int j = tid; j < ntok; j += DEC_THREADS) {
      uint32_t kc[W];
      if (j < copied) {
        if constexpr (W == 4) {
          uint4 v = reinterpret_cast<const uint4*>(st)[j];
          kc[0] = v.x; kc[1] = v.y; kc[2] = v.z; kc[3] = v.w;
        } else if constexpr (W == 8) {
          uint4 v0 = reinterpret_cast<const uint4*>(st)[2 * j], v1 = reinterpret_cast<const uint4*>(st)[2 * j + 1];
          kc[0] = v0.x; kc[1] = v0.y; kc[2] = v0.z; kc[3] = v0.w; kc[4] = v1.x; kc[5] = v1.y; kc[6] = v1.z; kc[7] = v1.w;
        } else {
#pragma unroll
          for (int w = 0; w < W; ++w) kc[w] = st[j * W + w];
        }
      } else {
        const uint32_t* gp = cbase + (t0 + base + j) * W;
#pragma unroll
        for (int w = 0; w < W; ++w) kc[w] = __ldg(gp + w);
      }
      const uint32_t D = group_distance<W, J>(kc, A, Bp);
      Dbuf[base + j] = (uint16_t)D;
      atomicAdd(&hist[D], 1u);
    }
    __syncthreads();
    if (tid == 0 && s + DEC_STAGES < nstages) issue_stage(s + DEC_STAGES);
  }

  // ---- phase 3: exact top-k' by counting select over the cluster (Alg. 3 lines 12-13)
  // threshold thr = D of the k'-th best token; all D < thr selected; ties at thr
  // selected lowest index first (R8) via per-CTA quotas in rank (= index) order.
  cluster.sync();                                                     // #1 histograms complete
  const int SL = (p.nbins + C - 1) / C;
  const int lo = r * SL, hi = min(p.nbins, lo + SL);
  const int nsl = hi > lo ? hi - lo : 0;
  for (int i = tid; i < SL + 1; i += DEC_THREADS) red[i] = 0;
  __syncthreads();
  for (int t = tid; t < nsl * C; t += DEC_THREADS) {
    const int i = t % nsl, c = t / nsl;
    const uint32_t* rh = cluster.map_shared_rank(hist, c);
    atomicAdd(&red[i], rh[lo + i]);
  }
  __syncthreads();
  if (warp == 0) {
    uint32_t sum = 0;
    for (int i = lane; i < nsl; i += 32) sum += red[i];
    sum = (uint32_t)warp_sum_i((int)sum);
    if (lane == 0) red[SL] = sum;                                     // slice total
  }
  cluster.sync();                                                     // #2 slice sums published
  if (warp == 0) {
    // locate the slice holding the k'-th smallest D
    uint32_t tot = 0;
    if (lane < C) tot = *cluster.map_shared_rank(red + SL, lane);
    uint32_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const uint32_t want = (uint32_t)kp;
    const uint32_t m = __ballot_sync(0xffffffffu, lane < C && incl >= want);
    int sstar = m ? __ffs(m) - 1 : 0;
    uint32_t before = __shfl_sync(0xffffffffu, incl - tot, sstar);
    // scan the slice's reduced bins
    const uint32_t* rr = cluster.map_shared_rank(red, sstar);
    const int slo = sstar * SL, snb = min(p.nbins, slo + SL) - slo;
    int thr = -1;
    uint32_t below = 0;
    for (int i0 = 0; i0 < snb && thr < 0; i0 += 32) {
      uint32_t v = (i0 + lane < snb) ? rr[i0 + lane] : 0u;
      uint32_t inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
      }
      const uint32_t mm = __ballot_sync(0xffffffffu, before + inc >= want && (i0 + lane < snb));
      if (mm) {
        const int l = __ffs(mm) - 1;
        thr = slo + i0 + l;
        below = __shfl_sync(0xffffffffu, before + inc - v, l);
      } else {
        before += __shfl_sync(0xffffffffu, inc, 31);
      }
    }
    if (kp == 0) { thr = -1; below = 0; }
    if (lane == 0) { misc[0] = thr; misc[1] = (int)below; }
  }
  __syncthreads();
  const int thr = misc[0];
  const int need = kp - misc[1];                                      // ties to take at thr
  // local: # tokens with D < thr, # ties at thr
  if (warp == 0) {
    uint32_t lt = 0;
    for (int i = lane; i < thr; i += 32) lt += hist[i];
    lt = (uint32_t)warp_sum_i((int)lt);
    if (lane == 0) { pub[0] = (int)lt; pub[1] = thr >= 0 ? (int)hist[thr] : 0; }
  }
  cluster.sync();                                                     // #3 (below_r, ties_r) published
  if (warp == 0) {
    int bl = 0, ti = 0;
    if (lane < C) { const int32_t* rp = cluster.map_shared_rank(pub, lane); bl = rp[0]; ti = rp[1]; }
    int incl = ti;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int tp = incl - ti;                                          // ties in lower ranks
    const int quota = max(0, min(need - tp, ti));
    const int contrib = (lane < r) ? bl + quota : 0;
    const int offset = warp_sum_i(contrib);
    const int myquota = __shfl_sync(0xffffffffu, quota, r);
    if (lane == 0) { misc[2] = offset; misc[3] = myquota; }
  }
  __syncthreads();
  const int offset_r = misc[2], quota_r = misc[3];
  const int R = (kp + C - 1) / C;                                     // rows per CTA for attention
  // order-preserving compaction: each warp owns a contiguous segment
  const int seg = ((Lr + DEC_WARPS - 1) / DEC_WARPS + 31) & ~31;
  const int s0 = min(Lr, warp * seg), s1 = min(Lr, s0 + seg);
  int lt_w = 0, ti_w = 0;
  for (int j0 = s0; j0 < s1; j0 += 32) {
    const int j = j0 + lane;
    const int Dv = j < s1 ? (int)Dbuf[j] : 0x7fffffff;
    lt_w += __popc(__ballot_sync(0xffffffffu, Dv < thr));
    ti_w += __popc(__ballot_sync(0xffffffffu, Dv == thr));
  }
  int* wcnt = misc + 8;                                               // [DEC_WARPS][2]
  if (lane == 0) { wcnt[2 * warp] = lt_w; wcnt[2 * warp + 1] = ti_w; }
  __syncthreads();
  int lt_b = 0, ti_b = 0;
  for (int w = 0; w < warp; ++w) { lt_b += wcnt[2 * w]; ti_b += wcnt[2 * w + 1]; }
  int32_t* oidx = p.out_idx ? p.out_idx + (int64_t)bg * p.k : nullptr;
  int32_t* osc = p.out_score ? p.out_score + (int64_t)bg * p.k : nullptr;
  int32_t* ocd = p.cand_D ? p.cand_D + (int64_t)bg * p.k : nullptr;
  const int Gr = G * p.rbits;
  for (int j0 = s0; j0 < s1; j0 += 32) {
    const int j = j0 + lane;
    const int Dv = j < s1 ? (int)Dbuf[j] : 0x7fffffff;
    const uint32_t lm = __ballot_sync(0xffffffffu, Dv < thr);
    const uint32_t tm = __ballot_sync(0xffffffffu, Dv == thr);
    const uint32_t below_me = (1u << lane) - 1u;
    const int my_tie_rank = ti_b + __popc(tm & below_me);
    const bool is_sel = (Dv < thr) || (Dv == thr && my_tie_rank < quota_r);
    if (is_sel) {
      const int lt_before = lt_b + __popc(lm & below_me);
      const int P = offset_r + lt_before + min(my_tie_rank, quota_r);
      const int tok = (int)(t0 + j);
      const int dest = P / R, slot = P - dest * R;
      if (p.gsel) p.gsel[((int64_t)bg * C + dest) * p.rows_cap + slot] = tok;
      else *cluster.map_shared_rank(sel + slot, dest) = tok;
      if (oidx) oidx[P] = (int32_t)(tok + p.token_offset);
      if (osc) osc[P] = Gr - 2 * Dv;                                   // S = G*rbits - 2D
      if (ocd) ocd[P] = Dv;
    }
    lt_b += __popc(lm);
    ti_b += __popc(tm);
  }
  if (r == 0) {
    for (int i = kp + tid; i < p.k; i += DEC_THREADS) {
      if (oidx) oidx[i] = -1;
      if (osc) osc[i] = 0;
      if (ocd) ocd[i] = 0x7fffffff;
    }
  }
  cluster.sync();                                                     // #4 selected lists complete

  if (p.cand_mode) {                                                  // sequence-shard phase 1 stops here
    cluster.sync();
    return;
  }
  cluster.sync();                                                     // #4 selected lists complete

  // ---- phase 4: gather + online-softmax attention over this CTA's rows (Alg. 3 lines 14-17)
  const int row0 = r * R;
  const int Rr = max(0, min(R, kp - row0));
  const T* Kb = reinterpret_cast<const T*>(p.K) + (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh;
  const T* Vb = reinterpret_cast<const T*>(p.V) + (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh;
  __syncthreads();                                                    // ring becomes attention scratch
  attend_rows<T, GT, D_HEAD>(sel, Rr, Kb, Vb, p.kv_st, qf, G, p.scale, reinterpret_cast<float*>(ring), part);
  cluster.sync();                                                     // #5 CTA partials published
  // ---- phase 5: combine the C partials in rank order (flash-decoding merge)
  cluster_combine<D_HEAD>(cluster, part, C, r, G, ((int64_t)b * p.Hq + g * G), p.out, p.out_bf16, nullptr);
  cluster.sync();                                                     // #6 keep smem alive for readers
}

// ---------------------------------------------------------------------------
// Sequence-shard phase 3: partial attention over this rank's selected rows.
struct PartialParams {
  const void* q;
  const void* K;
  const void* V;
  int64_t kv_sb, kv_sh, kv_st;
  const int32_t* own_idx;  // [B, Hkv, k] local row indices
  const int32_t* own_cnt;  // [B, Hkv]
  int B, Hq, Hkv, G, d, k;
  float scale;
  float* partial;          // [B, Hq, d+2]
  int C;
};

template <typename T, int GT, int D_HEAD>
__global__ void __launch_bounds__(DEC_THREADS, 1) hata_partial_attn_kernel(const __grid_constant__ PartialParams p) {
  extern __shared__ __align__(16) float psm[];
  cg::cluster_group cluster = cg::this_cluster();
  const int C = p.C, r = (int)cluster.block_rank();
  const int bg = blockIdx.y, b = bg / p.Hkv, g = bg % p.Hkv, G = p.G;
  float* qf = psm;                                  // [GT][d]
  float* part = qf + GT * D_HEAD;                   // [GT][d+2]
  float* wp = part + GT * (D_HEAD + 2);             // [DEC_WARPS][GT][d+2]
  const T* qg = reinterpret_cast<const T*>(p.q) + ((int64_t)b * p.Hq + (int64_t)g * G) * D_HEAD;
  for (int i = threadIdx.x; i < G * D_HEAD; i += DEC_THREADS) qf[i] = Elem<T>::to_f(qg[i]);
  const int cnt = p.own_cnt[bg];
  const int R = (cnt + C - 1) / C;
  const int Rr = max(0, min(R, cnt - r * R));
  __syncthreads();
  const T* Kb = reinterpret_cast<const T*>(p.K) + (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh;
  const T* Vb = reinterpret_cast<const T*>(p.V) + (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh;
  attend_rows<T, GT, D_HEAD>(p.own_idx + (int64_t)bg * p.k + (int64_t)r * R, Rr, Kb, Vb, p.kv_st, qf, G, p.scale,
                             wp, part);
  cluster.sync();
  cluster_combine<D_HEAD>(cluster, part, C, r, G, (int64_t)b * p.Hq + g * G, nullptr, 0, p.partial);
  cluster.sync();
}

}  // namespace hata
