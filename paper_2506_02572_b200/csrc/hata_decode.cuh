// Fused HATA decode kernel: q-hash -> Hamming score + GQA aggregate -> exact
// top-k (lowest index wins) -> gather + softmax attention -> split combine, in
// ONE launch.
//
// Work decomposition: a "unit" is one (b, KV head);
// each unit is served by M CTAs ("ranks") that own contiguous token chunks, so
// the grid (M x units) covers the 148 SMs even when B*H_kv is small.  The
// launch is cooperative (all CTAs co-resident) and the ranks of a unit meet
// exactly once, at a global-memory barrier after scoring, to exchange their
// D-histograms.  Every rank then derives the same threshold, per-rank tie
// quotas and output offsets, takes an equal share of the k' selected rows
// (re-scanning the D arrays it needs from L2), attends to them, and the last
// rank to finish merges the M softmax partials in rank order.
//
// PAPER: Alg. 3 lines 6, 10-17; §4.
// Readings R1-R20 are listed in DESIGN.md.
#pragma once
#include "hata_common.cuh"
#include "hata_score.cuh"

namespace hata {

constexpr int DEC_THREADS = 512;
constexpr int DEC_WARPS = DEC_THREADS / 32;
constexpr int DEC_STAGE_BYTES = 16384;       // one bulk copy of codes
constexpr int DEC_STAGES = 6;                // code ring depth (96 KB in flight)
constexpr int DEC_RING_BYTES = DEC_STAGE_BYTES * DEC_STAGES;
constexpr int DEC_D_SMEM_MAX = 16384;        // tokens/CTA whose D (u16) stays in smem
constexpr int DEC_CHUNK_ALIGN = 64;          // tokens
constexpr int DEC_MAX_RANKS = 32;            // M cap (histogram exchange is M x nbins per rank)
constexpr int DEC_ROW_PAD = 16;              // bytes of padding per staged K/V row (bank spread)
constexpr int DEC_QS_PAD = 4;                // floats of padding per q row in smem

struct DecodeParams {
  const void* q;           // [B, Hq, d] contiguous
  const void* K;           // caches, element strides, d contiguous
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
  // decomposition
  int M;                   // ranks (CTAs) per unit
  int chunk;               // tokens per rank (capacity), multiple of DEC_CHUNK_ALIGN
  int nbins;               // G*rbits + 1
  int rows_cap;            // rows per attention batch held in smem
  int R_cap;               // selected rows per rank (capacity of the rows list)
  int32_t* ws_rows;        // [units, M, R_cap] rows list when it does not fit in smem, else null
  int d_smem;              // 1: this rank's D lives in smem (mirrored to ws_D when M > 1)
  // workspace (global); zero-initialised once, left zeroed by every launch
  int32_t* ws_hist;        // [units, M, nbins]            (M > 1)
  uint16_t* ws_D;          // [units, M, chunk]            (M > 1 or !d_smem)
  float* ws_part;          // [units, M, GT, d+2]          (M > 1)
  unsigned* ws_sync;       // [units, 2]: barrier, done    (M > 1)
  // sequence-shard phase 1 (hata_shard_candidates): stop after the select and
  // emit (D, global index) candidates instead of attending.
  int cand_mode;
  int64_t token_offset;    // global index of local token 0
  int32_t* cand_D;         // [B, Hkv, k] or null
  // fused append (hata_decode_step): write k_new/v_new and the key code at row
  // n[b]-1 before scoring; null = caches already hold the new token
  const void* k_new;       // [B, Hkv, d]
  const void* v_new;
};

struct DecodeSmem {
  int ring, W, bars, hist, D, qf, qw, planes, rows, red, misc, total;
  int qp;                  // q-projection partial sums [DEC_THREADS/rbits][GT][rbits]
  int hm, kv, sc, rb;      // aliases inside ring+W after scoring
  int sc_limit;            // end of the reusable ring+W area
};

__host__ __device__ inline int dec_qstride(int d) { return d + DEC_QS_PAD; }
__host__ __device__ inline int dec_hist_stride(int nbins) { return (nbins + 3) & ~3; }
// floats per rank partial block [GT][d+2], padded to 16 bytes
__host__ __device__ inline int dec_part_stride(int GT, int d) { return (GT * (d + 2) + 3) & ~3; }

// Diagnostics: when non-null, CTA (x, y) writes globaltimer stamps of its
// phase boundaries to g_hata_trace[(y * gridDim.x + x) * 16 + i].  Set via
// hata_debug_trace(); null (off) by default.  One copy per translation unit.
static __device__ unsigned long long* g_hata_trace = nullptr;
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define HATA_TRACE(i)                                                                               \
  do {                                                                                              \
    if (g_hata_trace != nullptr && threadIdx.x == 0)                                                \
      g_hata_trace[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 16 + (i)] = globaltimer_ns();    \
  } while (0)

// Shared-memory carve-up; identical on host and device.
__host__ __device__ inline DecodeSmem decode_smem_layout(const DecodeParams& p, int GT, int eb) {
  auto up = [](int x) { return (x + 127) & ~127; };
  DecodeSmem s;
  int off = 0;
  s.ring = off; off += DEC_RING_BYTES;
  s.W = off; off += up(p.d * p.rbits * eb);
  s.bars = off; off += up((DEC_STAGES + 3) * 8);
  s.hist = off; off += up(p.nbins * 4);
  s.D = off; off += p.d_smem ? up(p.chunk * 2) : 0;
  s.qf = off; off += up((GT + 1) * dec_qstride(p.d) * 4);
  s.qw = off; off += up((GT + 1) * (p.rbits / 32) * 4);
  s.planes = off; off += up(2 * 4 * 8 * 4);
  s.rows = off; off += p.ws_rows ? 0 : up(p.R_cap * 4);
  s.red = off; off += up((DEC_MAX_RANKS * 4 + 64) * 4);
  s.misc = off; off += up(128 * 4);   // [0,16) scalars, [16,80) warp counters, [80,104) softmax m/l/corr
  s.qp = off; off += up(DEC_THREADS * (GT + 1) * 4);
  s.total = off;
  // after scoring the ring + W region is free:
  //   hm  : [M][nbins] int32 histograms of all ranks (select phase)
  //   kv  : staged K rows then V rows, [rows_cap][d*eb + pad] each (attention phase)
  //   sc  : [GT][rows_cap] fp32 logits / probabilities
  const int rowb = p.d * eb + DEC_ROW_PAD;
  s.hm = 0;
  s.kv = 0;
  s.sc = up(2 * p.rows_cap * rowb);
  s.rb = rowb;
  s.sc_limit = s.bars;
  return s;
}

// ----------------------------------------------------------------- helpers
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Order-preserving scan of one rank's D array (token order).  Tokens with
// D < thr are selected; ties (D == thr) are selected while their tie rank is
// below `quota`.  Each selected token gets position pos = base + #selected
// before it in this chunk; positions in [P0, P1) are emitted via `emit`.
// All threads of the block must call (block-uniform arguments).
// Vectorised: a lane owns 8 consecutive tokens (one 16-byte load), a warp a
// contiguous segment of 256-token blocks.  Dc must be 16-byte aligned.
template <typename Emit>
__device__ __forceinline__ void scan_chunk(const uint16_t* Dc, bool from_global, int L, int thr, int quota, int base,
                                           int P0, int P1, int* wcnt, Emit emit) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int seg = ((L + DEC_WARPS - 1) / DEC_WARPS + 255) & ~255;
  const int s0 = min(L, warp * seg), s1 = min(L, s0 + seg);
  // 8-bit masks of (D < thr) and (D == thr) for tokens j .. j+7
  auto masks = [&](int j, uint32_t& ltm, uint32_t& tim) {
    uint32_t v[4];
    if (j + 8 <= s1) {
      const uint4 x = from_global ? __ldcg(reinterpret_cast<const uint4*>(Dc + j))
                                  : *reinterpret_cast<const uint4*>(Dc + j);
      v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t lo = (j + 2 * e < s1) ? (uint32_t)(from_global ? __ldcg(Dc + j + 2 * e) : Dc[j + 2 * e]) : 0xffffu;
        const uint32_t hi = (j + 2 * e + 1 < s1) ? (uint32_t)(from_global ? __ldcg(Dc + j + 2 * e + 1) : Dc[j + 2 * e + 1])
                                                 : 0xffffu;
        v[e] = lo | (hi << 16);
      }
    }
    ltm = 0; tim = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int dv = (int)((v[e >> 1] >> (16 * (e & 1))) & 0xffffu);
      ltm |= (uint32_t)(dv < thr) << e;
      tim |= (uint32_t)(dv == thr) << e;
    }
  };
  int lt_w = 0, ti_w = 0;
  for (int j0 = s0; j0 < s1; j0 += 256) {
    uint32_t ltm = 0, tim = 0;
    if (j0 + 8 * lane < s1) masks(j0 + 8 * lane, ltm, tim);
    lt_w += __popc(ltm);
    ti_w += __popc(tim);
  }
  lt_w = warp_sum_i(lt_w);
  ti_w = warp_sum_i(ti_w);
  __syncthreads();                      // wcnt reuse guard
  if (lane == 0) { wcnt[2 * warp] = lt_w; wcnt[2 * warp + 1] = ti_w; }
  __syncthreads();
  int lt_b = 0, ti_b = 0;
  for (int w = 0; w < warp; ++w) { lt_b += wcnt[2 * w]; ti_b += wcnt[2 * w + 1]; }
  // skip whole segments whose positions fall outside [P0, P1) (warp-uniform)
  const int seg_first = base + lt_b + min(ti_b, quota);
  const int seg_last = base + lt_b + lt_w + min(ti_b + ti_w, quota);  // exclusive
  if (seg_last <= P0 || seg_first >= P1) return;
  for (int j0 = s0; j0 < s1; j0 += 256) {
    const int j = j0 + 8 * lane;
    uint32_t ltm = 0, tim = 0;
    if (j < s1) masks(j, ltm, tim);
    // warp-exclusive prefix of (lt, tie) counts, packed in one int
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
      if (((ltm >> e) & 1u) || tr < quota) {
        const int pos = base + ltl + __popc(ltm & below) + min(tr, quota);
        if (pos >= P0 && pos < P1) {
          const int dv = from_global ? (int)__ldcg(Dc + j + e) : (int)Dc[j + e];
          emit(pos, j + e, dv);
        }
      }
    }
    lt_b += tot & 0xffff;
    ti_b += tot >> 16;
  }
}

// Per-thread slice of the attention output: head h, elements 2*e2, 2*e2+1.
template <int GT, int D_HEAD>
struct AttnState {
  static constexpr int NSL = (GT * D_HEAD / 2 + DEC_THREADS - 1) / DEC_THREADS;  // slices per thread
  float acc[NSL][2];
};

// Softmax attention of the G heads over `Rr` rows whose cache indices are in
// rows[0..Rr) (smem), in batches of `rows_cap` rows staged in smem with
// cp.async -- the gather is fused into the attention: selected rows
// never land in HBM.  Logits: fp32 FMA over exact bf16 products; softmax and
// P.V in fp32 (R14).  On return: m_s[h], l_s[h] (smem, max logit and sum of
// exp) and st.acc (registers, this thread's unnormalised output slices).
template <typename T, int GT, int D_HEAD>
__device__ __forceinline__ void attend_rows(const int32_t* rows, int Rr, const T* __restrict__ Kb,
                                            const T* __restrict__ Vb, int64_t kv_st, const float* qf, int G,
                                            float scale, uint8_t* kvbuf, float* sc, int rows_cap, int rowb,
                                            float* m_s, float* l_s, float* corr_s, AttnState<GT, D_HEAD>& st) {
  constexpr int EB = sizeof(T);
  constexpr int CH = D_HEAD * EB / 16;          // 16-byte chunks per row
  constexpr int NSL = AttnState<GT, D_HEAD>::NSL;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int QS = dec_qstride(D_HEAD);
  uint8_t* Ks = kvbuf;
  uint8_t* Vs = kvbuf + rows_cap * rowb;
#pragma unroll
  for (int s = 0; s < NSL; ++s) st.acc[s][0] = st.acc[s][1] = 0.f;
  if (tid < GT) { m_s[tid] = -INFINITY; l_s[tid] = 0.f; }
  for (int r0 = 0; r0 < Rr; r0 += rows_cap) {
    const int nb = min(rows_cap, Rr - r0);
    __syncthreads();                            // previous batch fully consumed
    {
      // thread -> fixed (K|V, 16-byte chunk) column, strided over rows
      constexpr int CH2 = 2 * CH;
      static_assert(DEC_THREADS % CH2 == 0, "row stride");
      const int col = tid % CH2, which = col / CH, ch = col % CH;
      const T* base = (which ? Vb : Kb) + ch * (16 / EB);
      uint8_t* dst = (which ? Vs : Ks) + ch * 16;
      for (int i = tid / CH2; i < nb; i += DEC_THREADS / CH2)
        cp_async16(dst + i * rowb, base + (int64_t)rows[r0 + i] * kv_st);
    }
    cp_async_wait_all();
    __syncthreads();
    // logits z[h][i] = scale * q_h . K_i
    for (int pidx = tid; pidx < nb * GT; pidx += DEC_THREADS) {
      const int i = pidx % nb, h = pidx / nb;
      float z = 0.f;
      if (h < G) {
        const uint8_t* kr = Ks + i * rowb;
        const float* qh = qf + h * QS;
#pragma unroll 4
        for (int c = 0; c < CH; ++c) {
          float kv[16 / EB];
          if constexpr (EB == 2) {
            const uint4 raw = *reinterpret_cast<const uint4*>(kr + c * 16);
            const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
            for (int e = 0; e < 4; ++e) { float2 f = __bfloat1622float2(hh[e]); kv[2 * e] = f.x; kv[2 * e + 1] = f.y; }
          } else {
            const float4 raw = *reinterpret_cast<const float4*>(kr + c * 16);
            kv[0] = raw.x; kv[1] = raw.y; kv[2] = raw.z; kv[3] = raw.w;
          }
#pragma unroll
          for (int e = 0; e < 16 / EB; ++e) z = fmaf(qh[c * (16 / EB) + e], kv[e], z);
        }
        z *= scale;
      }
      sc[h * rows_cap + i] = z;
    }
    __syncthreads();
    // running max / rescale per head (warp h)
    for (int h = warp; h < G; h += DEC_WARPS) {
      float mb = -INFINITY;
      for (int i = lane; i < nb; i += 32) mb = fmaxf(mb, sc[h * rows_cap + i]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, o));
      const float mo = m_s[h];
      const float mn = fmaxf(mo, mb);
      float ls = 0.f;
      for (int i = lane; i < nb; i += 32) {
        const float pz = expf(sc[h * rows_cap + i] - mn);
        sc[h * rows_cap + i] = pz;
        ls += pz;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o);
      if (lane == 0) {
        const float cr = (mo == -INFINITY) ? 0.f : expf(mo - mn);
        corr_s[h] = cr;
        l_s[h] = l_s[h] * cr + ls;
        m_s[h] = mn;
      }
    }
    __syncthreads();
    // acc[h][e] = corr * acc + sum_i p[h][i] * V[i][e]
#pragma unroll
    for (int s = 0; s < NSL; ++s) {
      const int sl = tid + s * DEC_THREADS;
      const int h = sl / (D_HEAD / 2), e2 = sl % (D_HEAD / 2);
      if (h < G) {
        const float cr = corr_s[h];
        float a0 = st.acc[s][0] * cr, a1 = st.acc[s][1] * cr;
        const float* ph = sc + h * rows_cap;
#pragma unroll 4
        for (int i = 0; i < nb; ++i) {
          float v0, v1;
          if constexpr (EB == 2) {
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(Vs + i * rowb + e2 * 4));
            v0 = f.x; v1 = f.y;
          } else {
            const float2 f = *reinterpret_cast<const float2*>(Vs + i * rowb + e2 * 8);
            v0 = f.x; v1 = f.y;
          }
          const float pz = ph[i];
          a0 = fmaf(pz, v0, a0);
          a1 = fmaf(pz, v1, a1);
        }
        st.acc[s][0] = a0; st.acc[s][1] = a1;
      }
    }
  }
  __syncthreads();
}

// Projection of one fp32 vector x[d] (smem) onto 32 consecutive hash bits
// [bit0, bit0+32) of W_g (smem), one packed word (lane i -> bit i).
// Alg. 2: Sign(MatMul) then BitPack, LSB-first; sign(0) -> 1.
template <typename T>
__device__ __forceinline__ uint32_t hash_word_smem(const float* __restrict__ x, const T* __restrict__ Ws, int d,
                                                   int rbits, int bit0, int lane) {
  float a0 = 0.f, a1 = 0.f;
  const T* col = Ws + bit0 + lane;
#pragma unroll 8
  for (int j = 0; j < d; j += 2) {
    a0 = fmaf(x[j], Elem<T>::to_f(col[j * rbits]), a0);
    a1 = fmaf(x[j + 1], Elem<T>::to_f(col[(j + 1) * rbits]), a1);
  }
  return __ballot_sync(0xffffffffu, (a0 + a1) >= 0.f);
}

template <typename T, int W, int GT, int D_HEAD>
__global__ void __launch_bounds__(DEC_THREADS, 1) hata_decode_kernel(const __grid_constant__ DecodeParams p) {
  constexpr int J = planes_for_group(GT);
  constexpr int STAGE_TOK = DEC_STAGE_BYTES / (W * 4);
  constexpr int EB = sizeof(T);
  constexpr int NSL = AttnState<GT, D_HEAD>::NSL;
  extern __shared__ __align__(1024) uint8_t smem[];

  const int M = p.M;
  const int r = blockIdx.x;
  const int u = blockIdx.y;
  const int b = u / p.Hkv, g = u % p.Hkv;
  const int G = p.G;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const DecodeSmem L = decode_smem_layout(p, GT, EB);
  const int QS = dec_qstride(D_HEAD);

  uint8_t* ring = smem + L.ring;
  T* Ws = reinterpret_cast<T*>(smem + L.W);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
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

  const int64_t n = p.n[b];
  const int kp = (int)(n < (int64_t)p.k ? n : (int64_t)p.k);      // k' = min(k, n)  (R10)
  // rank chunks [rr*per, (rr+1)*per) of this sequence
  int per = (int)(((n + M - 1) / M + DEC_CHUNK_ALIGN - 1) / DEC_CHUNK_ALIGN * DEC_CHUNK_ALIGN);
  if (per > p.chunk) per = p.chunk;
  if (per < DEC_CHUNK_ALIGN) per = DEC_CHUNK_ALIGN;
  auto chunk_len = [&](int rr) -> int {
    const int64_t a = (int64_t)rr * per, z = min((int64_t)n, a + per);
    return z > a ? (int)(z - a) : 0;
  };
  const int64_t t0 = (int64_t)r * per;
  const int Lr = chunk_len(r);
  const int nstages = (Lr + STAGE_TOK - 1) / STAGE_TOK;
  const uint32_t* cbase = p.codes + (int64_t)b * p.c_sb + (int64_t)g * p.c_sh;

  // ---- phase 0: start the code stream and the W_g copy (both q-independent)
  if (tid == 0) {
    // code ring [0, STAGES), W copy [STAGES], histogram/D staging [STAGES + 1], partials [STAGES + 2]
    for (int s = 0; s < DEC_STAGES + 3; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue_stage = [&](int s) {
    const int slot = s % DEC_STAGES;
    const int ntok = min(STAGE_TOK, Lr - s * STAGE_TOK);
    const uint32_t bytes = (uint32_t)(ntok * W * 4) & ~15u;
    mbar_arrive_expect_tx(&bars[slot], bytes);
    if (bytes) bulk_g2s(ring + slot * DEC_STAGE_BYTES, cbase + (t0 + (int64_t)s * STAGE_TOK) * W, bytes, &bars[slot]);
  };
  if (tid == 0) {
    const uint32_t wbytes = (uint32_t)(p.d * p.rbits * EB);
    mbar_arrive_expect_tx(&bars[DEC_STAGES], wbytes);
    bulk_g2s(Ws, reinterpret_cast<const T*>(p.Wh) + (int64_t)g * p.d * p.rbits, wbytes, &bars[DEC_STAGES]);
    for (int s = 0; s < DEC_STAGES && s < nstages; ++s) issue_stage(s);
  }
  for (int i = tid; i < p.nbins; i += DEC_THREADS) hist[i] = 0;

  HATA_TRACE(0);
  // ---- phase 1: Encode & Cache update (Alg. 3 lines 2-9; fused as
  // in §4): hash the G query heads of the group and, when this launch
  // also appends the new token (k_new != null), its key -- one projection pass
  // with the key as row G.  The rank owning row pos = n-1 writes K/V/code rows.
  const int64_t pos = n - 1;
  const bool append = p.k_new != nullptr && n >= 1;
  const bool owner = append && pos >= t0 && pos < t0 + Lr;
  const int NV = G + (owner ? 1 : 0);                                // projected vectors
  const T* qg = reinterpret_cast<const T*>(p.q) + ((int64_t)b * p.Hq + (int64_t)g * G) * D_HEAD;
  for (int i = tid; i < G * D_HEAD; i += DEC_THREADS) qf[(i / D_HEAD) * QS + i % D_HEAD] = Elem<T>::to_f(qg[i]);
  if (owner) {
    const T* kn = reinterpret_cast<const T*>(p.k_new) + (int64_t)u * D_HEAD;
    const T* vn = reinterpret_cast<const T*>(p.v_new) + (int64_t)u * D_HEAD;
    T* Kd = const_cast<T*>(reinterpret_cast<const T*>(p.K)) + (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh + pos * p.kv_st;
    T* Vd = const_cast<T*>(reinterpret_cast<const T*>(p.V)) + (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh + pos * p.kv_st;
    for (int i = tid; i < D_HEAD; i += DEC_THREADS) {
      const T kv = kn[i];
      Kd[i] = kv;                                                      // Alg. 3 line 3
      Vd[i] = vn[i];                                                   // Alg. 3 line 4
      qf[G * QS + i] = Elem<T>::to_f(kv);
    }
  }
  __syncthreads();
  mbar_wait(&bars[DEC_STAGES], 0);
  {
    // projection p[h][bit] = sum_j x_h[j] W[j][bit]: thread = (bit, j-slice), all
    // vectors at once; slices summed in fixed order (fp32 accumulation, R13)
    float* qpart = reinterpret_cast<float*>(smem + L.qp);           // [nparts][GT+1][rbits]
    const int nparts = DEC_THREADS / p.rbits;
    const int bit = tid % p.rbits, part = tid / p.rbits;           // part is warp-uniform
    const int jlen = D_HEAD / nparts;
    float acc[GT + 1];
#pragma unroll
    for (int h = 0; h <= GT; ++h) acc[h] = 0.f;
    const T* wc = Ws + bit;
    for (int j0 = part * jlen; j0 < (part + 1) * jlen; j0 += 4) {
      float wv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) wv[e] = Elem<T>::to_f(wc[(j0 + e) * p.rbits]);
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
    // Sign + BitPack (Alg. 2 lines 5-7): a warp covers 32 consecutive bits of one vector
    for (int o = tid; o < NV * p.rbits; o += DEC_THREADS) {
      const int h = o / p.rbits, bb = o % p.rbits;
      float sum = 0.f;
      for (int pp = 0; pp < nparts; ++pp) sum += qpart[(pp * (GT + 1) + h) * p.rbits + bb];
      const uint32_t word = __ballot_sync(0xffffffffu, sum >= 0.f);
      if (lane == 0) {
        qw[h * W + bb / 32] = word;                                    // row G = new key code
        if (h < G && p.out_qcodes && r == 0) p.out_qcodes[((int64_t)b * p.Hq + g * G + h) * W + bb / 32] = word;
        if (h == G)                                                    // Alg. 3 line 9
          const_cast<uint32_t*>(p.codes)[(int64_t)b * p.c_sb + (int64_t)g * p.c_sh + pos * W + bb / 32] = word;
      }
    }
  }
  __syncthreads();
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
  for (int s = 0; s < nstages; ++s) {
    const int slot = s % DEC_STAGES;
    mbar_wait(&bars[slot], (s / DEC_STAGES) & 1);
    const int ntok = min(STAGE_TOK, Lr - s * STAGE_TOK);
    const int copied = (int)(((uint32_t)(ntok * W * 4) & ~15u) / (W * 4));
    const uint32_t* st = reinterpret_cast<const uint32_t*>(ring + slot * DEC_STAGE_BYTES);
    const int base = s * STAGE_TOK;
    // two tokens per thread per iteration -> one 32-bit store of a u16 pair
    for (int j2 = tid; 2 * j2 < ntok; j2 += DEC_THREADS) {
      uint32_t Dpair[2];
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const int j = 2 * j2 + x;
        uint32_t kc[W];
#pragma unroll
        for (int w = 0; w < W; ++w) kc[w] = 0;
        if (j < copied) {
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
        } else if (j < ntok) {
          const uint32_t* gp = cbase + (t0 + base + j) * W;
#pragma unroll
          for (int w = 0; w < W; ++w) kc[w] = __ldg(gp + w);
        }
        if (j < ntok) {
          Dpair[x] = group_distance<W, J>(kc, A, Bp);
          atomicAdd(&hist[Dpair[x]], 1u);
        } else {
          Dpair[x] = 0xffffu;
        }
      }
      const uint32_t packed = Dpair[0] | (Dpair[1] << 16);
      reinterpret_cast<uint32_t*>(Dloc + base)[j2] = packed;
      if (mirror) reinterpret_cast<uint32_t*>(Dglob + base)[j2] = packed;
    }
    __syncthreads();
    if (tid == 0 && s + DEC_STAGES < nstages) issue_stage(s + DEC_STAGES);
  }
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
  // threshold thr = D of the k'-th best token; all D < thr are selected; ties
  // at thr are selected lowest index first (R8) via per-rank quotas in rank
  // (= token) order.  The ranks of a unit exchange histograms once.
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
      while (ld_acquire_gpu(sync) < (unsigned)M) {
      }
      // other ranks' generic-proxy writes -> this thread's async-proxy (bulk copy) reads
      asm volatile("fence.proxy.async.global;" ::: "memory");
      const uint32_t bytes = (uint32_t)(M * hs * 4);
      mbar_arrive_expect_tx(&bars[DEC_STAGES + 1], bytes);
      bulk_g2s(hm, p.ws_hist + (int64_t)u * M * hs, bytes, &bars[DEC_STAGES + 1]);
    }
    mbar_wait(&bars[DEC_STAGES + 1], 0);
  } else {
    for (int i = tid; i < p.nbins; i += DEC_THREADS) hm[i] = (int32_t)hist[i];
    __syncthreads();
  }
  HATA_TRACE(3);
  // total histogram (reuse `hist`)
  for (int i = tid; i < p.nbins; i += DEC_THREADS) {
    int s = 0;
    for (int rr = 0; rr < M; ++rr) s += hm[rr * hs + i];
    hist[i] = (uint32_t)s;
  }
  __syncthreads();
  if (warp == 0) {
    int before = 0, thr = -1, below = 0;
    for (int i0 = 0; i0 < p.nbins && thr < 0; i0 += 32) {
      const int v = (i0 + lane < p.nbins) ? (int)hist[i0 + lane] : 0;
      int inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int w2 = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += w2;
      }
      const uint32_t mm = __ballot_sync(0xffffffffu, before + inc >= kp && (i0 + lane < p.nbins));
      if (mm) {
        const int l = __ffs(mm) - 1;
        thr = i0 + l;
        below = __shfl_sync(0xffffffffu, before + inc - v, l);
      } else {
        before += __shfl_sync(0xffffffffu, inc, 31);
      }
    }
    if (kp <= 0) { thr = -1; below = 0; }
    if (lane == 0) { misc[0] = thr; misc[1] = kp - below; }
  }
  __syncthreads();
  const int thr = misc[0];
  const int need = misc[1];
  // per-rank (below, ties): warp w handles ranks w, w+8, ...
  int32_t* rb_below = red;                       // [M]
  int32_t* rb_ties = red + DEC_MAX_RANKS;        // [M]
  int32_t* rb_off = red + 2 * DEC_MAX_RANKS;     // [M]
  int32_t* rb_quota = red + 3 * DEC_MAX_RANKS;   // [M]
  for (int rr = warp; rr < M; rr += DEC_WARPS) {
    int s = 0;
    for (int i = lane; i < thr; i += 32) s += hm[rr * hs + i];
    s = warp_sum_i(s);
    if (lane == 0) { rb_below[rr] = s; rb_ties[rr] = thr >= 0 ? hm[rr * hs + thr] : 0; }
  }
  __syncthreads();
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
    if (lane < M) { rb_quota[lane] = quota; rb_off[lane] = inc2 - sel; }
  }
  __syncthreads();

  // this rank's equal share of the ascending selection: positions [P0, P1)
  const int R = (kp + M - 1) / M;
  const int P0 = min(kp, r * R), P1 = min(kp, P0 + R);
  int32_t* oidx = p.out_idx ? p.out_idx + (int64_t)u * p.k : nullptr;
  int32_t* osc = p.out_score ? p.out_score + (int64_t)u * p.k : nullptr;
  int32_t* ocd = p.cand_D ? p.cand_D + (int64_t)u * p.k : nullptr;
  const int Gr = G * p.rbits;
  int* wcnt = misc + 16;                         // [DEC_WARPS][2]
  // stage the D arrays of the other ranks whose selections overlap [P0, P1)
  // into smem with one bulk copy each (the ring + W area is free by now)
  int32_t* dslot = red + 4 * DEC_MAX_RANKS;      // [M] smem byte offset of rank c's D copy, -1 if none
  if (tid == 0) {
    asm volatile("fence.proxy.async.global;" ::: "memory");   // D written by generic stores
    uint32_t soff = (uint32_t)((M * hs * 4 + 127) & ~127), tx = 0;
    for (int c = 0; c < M; ++c) {
      dslot[c] = -1;
      const int off = rb_off[c], cnt = rb_below[c] + rb_quota[c];
      if (P1 <= P0 || cnt == 0 || off + cnt <= P0 || off >= P1) continue;
      if (c == r && p.d_smem) continue;
      const uint32_t bytes = (uint32_t)((chunk_len(c) * 2 + 15) & ~15);
      if (soff + bytes > (uint32_t)L.sc_limit) continue;          // does not fit: scan from L2
      dslot[c] = (int)soff;
      tx += bytes;
      soff += (bytes + 127) & ~127u;
    }
    if (tx) {
      mbar_arrive_expect_tx(&bars[DEC_STAGES + 1], tx);
      for (int c = 0; c < M; ++c)
        if (dslot[c] >= 0)
          bulk_g2s(smem + dslot[c], p.ws_D + ((int64_t)u * M + c) * p.chunk,
                   (uint32_t)((chunk_len(c) * 2 + 15) & ~15), &bars[DEC_STAGES + 1]);
    }
    misc[3] = tx ? 1 : 0;
  }
  __syncthreads();
  if (misc[3]) mbar_wait(&bars[DEC_STAGES + 1], M > 1 ? 1 : 0);
  HATA_TRACE(4);
  for (int c = 0; c < M && P1 > P0; ++c) {
    const int off = rb_off[c], cnt = rb_below[c] + rb_quota[c];
    if (cnt == 0 || off + cnt <= P0 || off >= P1) continue;    // block-uniform
    const bool own = (c == r) && p.d_smem;
    const bool staged = dslot[c] >= 0;
    const bool fromg = !own && !staged;
    const uint16_t* Dc = own ? Dloc
                             : (staged ? reinterpret_cast<const uint16_t*>(smem + dslot[c])
                                       : p.ws_D + ((int64_t)u * M + c) * p.chunk);
    const int64_t ctok = (int64_t)c * per;
    scan_chunk(Dc, fromg, chunk_len(c), thr, rb_quota[c], off, P0, P1, wcnt, [&](int pos, int j, int Dv) {
      const int tok = (int)(ctok + j);
      rows[pos - P0] = tok;
      if (oidx) oidx[pos] = (int32_t)(tok + p.token_offset);
      if (osc) osc[pos] = Gr - 2 * Dv;                       // S = G*rbits - 2D
      if (ocd) ocd[pos] = Dv;
    });
  }
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
    float* sc = reinterpret_cast<float*>(smem + L.sc);
    attend_rows<T, GT, D_HEAD>(rows, P1 - P0, Kb, Vb, p.kv_st, qf, G, p.scale, smem + L.kv, sc, p.rows_cap, L.rb,
                               m_s, l_s, corr_s, st);
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
  float* mypart = p.ws_part + ((int64_t)u * M + r) * dec_part_stride(GT, D_HEAD);
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
  if (!misc[2]) return;
  // last rank: all other partials are visible (their fence + the counter);
  // pull them into smem with one bulk copy, then merge in rank order
  if (!p.cand_mode) {
    const int PB = dec_part_stride(GT, D_HEAD);
    float* sp = reinterpret_cast<float*>(smem);                      // ring+W area is free
    if (tid == 0) {
      __threadfence();
      asm volatile("fence.proxy.async.global;" ::: "memory");
      const uint32_t bytes = (uint32_t)(M * PB * 4);
      mbar_arrive_expect_tx(&bars[DEC_STAGES + 2], bytes);
      bulk_g2s(sp, p.ws_part + (int64_t)u * M * PB, bytes, &bars[DEC_STAGES + 2]);
    }
    mbar_wait(&bars[DEC_STAGES + 2], 0);
    for (int o = tid; o < G * D_HEAD; o += DEC_THREADS) {
      const int h = o / D_HEAD, e = o % D_HEAD;
      float Mx = -INFINITY;
      for (int rr = 0; rr < M; ++rr) Mx = fmaxf(Mx, sp[rr * PB + h * PS]);
      float Ls = 0.f, As = 0.f;
      for (int rr = 0; rr < M; ++rr) {
        const float* pr = sp + rr * PB + h * PS;
        const float mr = pr[0];
        const float scl = (mr == -INFINITY) ? 0.f : expf(mr - Mx);
        Ls = fmaf(pr[1], scl, Ls);
        As = fmaf(pr[2 + e], scl, As);
      }
      store_out(h, e, Ls > 0.f ? As / Ls : 0.f);
    }
  }
  if (tid == 0) { sync[0] = 0u; sync[1] = 0u; }     // leave the workspace zeroed for the next launch
  HATA_TRACE(7);
}

// ---------------------------------------------------------------------------
// Sequence-shard phase 3: attention over this rank's selected rows -> raw
// (m, l, acc) partials.  One CTA per (b, KV head); rows in smem batches.
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
  int rows_cap;            // rows per smem batch
};

template <typename T, int GT, int D_HEAD>
__global__ void __launch_bounds__(DEC_THREADS, 1) hata_partial_attn_kernel(const __grid_constant__ PartialParams p) {
  extern __shared__ __align__(1024) uint8_t psm[];
  constexpr int EB = sizeof(T);
  constexpr int NSL = AttnState<GT, D_HEAD>::NSL;
  const int u = blockIdx.x, b = u / p.Hkv, g = u % p.Hkv, G = p.G;
  const int tid = threadIdx.x;
  const int QS = dec_qstride(D_HEAD);
  const int rowb = D_HEAD * EB + DEC_ROW_PAD;
  uint8_t* kv = psm;                                                         // [2][rows_cap][rowb]
  float* sc = reinterpret_cast<float*>(psm + ((2 * p.rows_cap * rowb + 127) & ~127));   // [GT][rows_cap]
  float* qf = sc + GT * p.rows_cap;                                          // [GT][QS]
  float* fm = qf + GT * QS;                                                  // m, l, corr
  int32_t* rows = reinterpret_cast<int32_t*>(fm + 32);                       // [k]
  const T* qg = reinterpret_cast<const T*>(p.q) + ((int64_t)b * p.Hq + (int64_t)g * G) * D_HEAD;
  for (int i = tid; i < G * D_HEAD; i += DEC_THREADS) qf[(i / D_HEAD) * QS + i % D_HEAD] = Elem<T>::to_f(qg[i]);
  const int cnt = p.own_cnt[u];
  for (int i = tid; i < cnt; i += DEC_THREADS) rows[i] = p.own_idx[(int64_t)u * p.k + i];
  __syncthreads();
  const T* Kb = reinterpret_cast<const T*>(p.K) + (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh;
  const T* Vb = reinterpret_cast<const T*>(p.V) + (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh;
  AttnState<GT, D_HEAD> st;
  float* m_s = fm;
  float* l_s = fm + 8;
  float* corr_s = fm + 16;
  attend_rows<T, GT, D_HEAD>(rows, cnt, Kb, Vb, p.kv_st, qf, G, p.scale, kv, sc, p.rows_cap, rowb, m_s, l_s, corr_s,
                             st);
  const int PS = D_HEAD + 2;
#pragma unroll
  for (int s = 0; s < NSL; ++s) {
    const int sl = tid + s * DEC_THREADS;
    const int h = sl / (D_HEAD / 2), e2 = sl % (D_HEAD / 2);
    if (h < G) {
      float* pr = p.partial + ((int64_t)b * p.Hq + g * G + h) * PS;
      pr[2 + 2 * e2] = st.acc[s][0];
      pr[3 + 2 * e2] = st.acc[s][1];
    }
  }
  if (tid < G) {
    float* pr = p.partial + ((int64_t)b * p.Hq + g * G + tid) * PS;
    pr[0] = m_s[tid];
    pr[1] = l_s[tid];
  }
}

}  // namespace hata
