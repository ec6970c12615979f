// Fused HATA decode kernel: q-hash -> Hamming score + GQA aggregate -> exact
// top-k (lowest index wins) -> gather + softmax attention -> split combine, in
// ONE launch.
//
// Work decomposition: a "unit" is one (b, KV head);
// each unit is served by M CTAs ("ranks") that own contiguous token chunks, so
// the grid (M x units) covers the 148 SMs even when B*H_kv is small.  The grid
// never exceeds one CTA per SM (co-resident once the SMs are free) and the
// ranks of a unit exchange data twice, through epoch-tagged 64-bit words in
// the workspace that the readers poll (no fences, no counters): the
// D-histogram prefix counts after scoring -- every rank then derives the same
// threshold, its own tie quota and output offset, compacts its OWN selected
// tokens in token order and attends to them -- and the softmax partials,
// merged in rank order by min(G, M) merger ranks (one or more heads each).
//
// PAPER: Alg. 3 lines 6, 10-17; §4.
// Readings R1-R20 are listed in DESIGN.md.
#pragma once
#include "hata_common.cuh"
#include "hata_score.cuh"

namespace hata {

#ifndef HATA_DEC_THREADS
#define HATA_DEC_THREADS 256
#endif
constexpr int DEC_THREADS = HATA_DEC_THREADS;
constexpr int DEC_WARPS = DEC_THREADS / 32;
constexpr int DEC_STAGE_BYTES = 32768;       // one bulk copy of codes (few large TMA requests)
constexpr int DEC_MAX_STAGES = 4;            // code ring depth (up to 128 KB in flight)
constexpr int DEC_D_SMEM_MAX = 16384;        // tokens/CTA whose D (u16) stays in smem
constexpr int DEC_CHUNK_ALIGN = 64;          // tokens
constexpr int DEC_BC_WPT = 4;               // candidate-bitmap words per thread (fast selection path)
#ifndef HATA_HINT_SLACK
#define HATA_HINT_SLACK 10  // measured (CFG-4, q varying): 2 -> 77 % hinted selections, 6 -> 98 %, 10 -> 100 % (17.84 -> 17.45 -> 17.30 us)
#endif
constexpr int DEC_HINT_SLACK = HATA_HINT_SLACK;   // hint threshold slack (bins)
constexpr int DEC_WIN = 32;                 // bins [h - 15, h + 16] (h = previous threshold) of every rank's prefix counts
constexpr int DEC_SYNC_WORDS = 8;            // per-unit sync words in the workspace
constexpr int DEC_MAX_RANKS = 32;            // M cap (histogram exchange is M x nbins per rank)
constexpr int DEC_ROW_PAD = 16;              // bytes of padding per staged K/V row (bank spread)
constexpr int DEC_QS_PAD = 4;                // floats of padding per q row in smem
// spin-wait rounds before a kernel traps instead of hanging (~seconds)
#ifndef HATA_SPIN_LIMIT
#define HATA_SPIN_LIMIT (1u << 24)
#endif

// Element (or word) offset of token t's row for one (b, KV head): contiguous
// caches (pt == null): base + t * st with base = b * sb + g * sh; paged caches
// (NEXT-2, P:260 serving engines): page table row pt of sequence b, rows of a
// physical page ps = 2^lg apart: pt[t >> lg] * sp + base + (t & (ps-1)) * st
// with base = g * sh.
struct RowMap {
  const int32_t* pt;
  int lg;
  int64_t sp, base, st;
  __device__ __forceinline__ int64_t operator()(int64_t t) const {
    return pt ? (int64_t)__ldg(pt + (t >> lg)) * sp + base + (t & ((1 << lg) - 1)) * st : base + t * st;
  }
};

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
  int stages;              // code ring stages (<= DEC_MAX_STAGES)
  int chunk;               // tokens per rank (capacity), multiple of DEC_CHUNK_ALIGN
  int nbins;               // G*rbits + 1
  int rows_cap;            // rows per attention batch held in smem
  int R_cap;               // selected rows per rank (capacity of the rows list) = min(k', chunk)
  int32_t* ws_rows;        // [units, M, R_cap] rows list when it does not fit in smem, else null
  int d_smem;              // 1: this rank's D lives in smem, else in ws_D
  // workspace (global); zero-initialised once, left zeroed by every launch
  // tagged words (tag << 32 | 32-bit value): tag = this launch's epoch, so a
  // reader that sees the tag sees the value -- no fences, no arrival counters
  uint64_t* ws_hist;       // [units, M, hs] exclusive prefix counts cum_r[0..nbins]   (M > 1)
  uint16_t* ws_D;          // [units, M, chunk] D when it does not fit in smem (!d_smem)
  uint64_t* ws_part;       // [units, M, GT, d+2] float bits  (M > 1)
  unsigned* ws_sync;       // [units, 8]: epoch, threshold hint (2 slots by epoch parity), hint-use counters,
                           //   appended row + 1 (2 slots by epoch parity), 2 spare
  // sequence-shard phase 1 (hata_shard_candidates): stop after the select and
  // emit (D, global index) candidates instead of attending.
  int cand_mode;
  int64_t token_offset;    // global index of local token 0
  int64_t n_max;           // host bound on n[b]: fixes the rank chunks (chunk = ceil(n_max/M)); n[b] is clamped to it
  int64_t cap;             // rows allocated per (b, KV head): the fused append writes row n-1 only if < cap
  int32_t* cand_D;         // [B, Hkv, k] or null
  // fused append (hata_decode_step): write k_new/v_new and the key code at row
  // n[b]-1 before scoring; null = caches already hold the new token
  const void* k_new;       // [B, Hkv, d]
  const void* v_new;
  // paged caches (hata_decode_step_paged): logical token t of sequence b is
  // slot t & (2^page_lg - 1) of physical page page_table[b * max_pages +
  // (t >> page_lg)]; kv_sb / c_sb are then the page strides.  null = contiguous
  const int32_t* page_table;
  int max_pages, page_lg;
  unsigned long long* trace;   // diagnostics (hata_debug_trace), null = off
  int dbg;                     // diagnostics: HATA_DEBUG bits (0 in production)
  int use_hint;                // threshold hint from the previous launch (HATA_HINT=0 disables)
};

struct DecodeSmem {
  int ring, W, bars, hist, D, bc, qf, qw, planes, rows, red, misc, chref, total;
  int qp;                  // q-projection partial sums [DEC_THREADS/rbits][GT][rbits]
  int qraw;                // q rows (+ the new key) as stored, bulk-copied
  int hm, kv, sc, rb;      // aliases inside ring+W after scoring
  int sc_limit;            // end of the reusable ring+W area
};

__host__ __device__ inline int dec_qstride(int d) { return d + DEC_QS_PAD; }
// tokens of a rank's D buffer: the chunk rounded up to 8 * DEC_THREADS (the
// selection reads whole uint4 blocks of 8 tokens per thread)
__host__ __device__ inline int dec_dchunk(int chunk) { return (chunk + 8 * DEC_THREADS - 1) / (8 * DEC_THREADS) * (8 * DEC_THREADS); }
__host__ __device__ inline int dec_hist_stride(int nbins) { return (nbins + 3) & ~3; }
// bytes of one W_g row in smem: padded by 16 so that 8 consecutive rows of a
// ldmatrix tile fall in distinct banks
__host__ __device__ inline int dec_wrow_stride(int rbits, int eb) { return rbits * eb + 16; }
// floats per rank partial block [GT][d+2], padded to 16 bytes
__host__ __device__ inline int dec_part_stride(int GT, int d) { return (GT * (d + 2) + 3) & ~3; }

// Diagnostics: when p.trace is non-null, CTA (x, y) writes globaltimer stamps
// of its phase boundaries to p.trace[(y * gridDim.x + x) * 16 + i].  Set via
// hata_debug_trace(); null (off) by default.  The pointer is a kernel
// parameter (constant bank), so the disabled check costs no memory access.
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
constexpr int HATA_TRACE_SLOTS = 96;   // [0, 32) %globaltimer stamps, [32, 64) clock64 stamps (HATA_CLK),
                                       // [64, 96) clock64 at the %globaltimer stamps
__device__ __forceinline__ void trace_at(unsigned long long* tr, int i) {
  if (tr != nullptr && threadIdx.x == 0) {
    unsigned long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)::"memory");
    const size_t base = ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * HATA_TRACE_SLOTS;
    tr[base + i] = globaltimer_ns();
    tr[base + 64 + i] = c;
  }
}
__device__ __forceinline__ void clock_at(unsigned long long* tr, int i) {
  if (tr != nullptr && threadIdx.x == 0) {
    unsigned long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)::"memory");
    tr[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * HATA_TRACE_SLOTS + 32 + i] = c;
  }
}
// Stamps are compiled in only for the diagnostics build (libhata_trace.so,
// HATA_TRACE_ENABLED=1); the production kernel carries none of this code.
#ifndef HATA_TRACE_ENABLED
#define HATA_TRACE_ENABLED 0
#endif
#define HATA_DIAG HATA_TRACE_ENABLED
#if HATA_TRACE_ENABLED
#define HATA_TRACE(i) trace_at(p.trace, (i))
#define HATA_CLK(i) clock_at(p.trace, (i))
#define HATA_TRACE_AT(tr, i) trace_at((tr), (i))
#else
#define HATA_TRACE(i) ((void)0)
#define HATA_CLK(i) ((void)0)
#define HATA_TRACE_AT(tr, i) ((void)0)
#endif

// Shared-memory carve-up; identical on host and device.
__host__ __device__ inline DecodeSmem decode_smem_layout(const DecodeParams& p, int GT, int eb) {
  auto up = [](int x) { return (x + 127) & ~127; };
  DecodeSmem s;
  int off = 0;
  s.ring = off; off += p.stages * DEC_STAGE_BYTES;
  s.W = off; off += up(p.d * dec_wrow_stride(p.rbits, eb));
  s.bars = off; off += up((DEC_MAX_STAGES + 4) * 8);
  s.hist = off; off += up(p.nbins * 4);
  s.D = off; off += p.d_smem ? up(dec_dchunk(p.chunk) * 2) : 0;
  s.bc = off; off += p.d_smem ? up(dec_dchunk(p.chunk) / 8) : 0;   // candidate bitmap (1 bit per token)
  s.qf = off; off += up((GT + 1) * dec_qstride(p.d) * 4);
  s.qw = off; off += up((GT + 2) * (p.rbits / 32) * 4);   // q codes, new key code, reloaded row
  s.qraw = off; off += up((GT + 2) * p.d * eb);   // q rows, new key, new value
  s.planes = off; off += up((64 + 8) * 4);        // P/N planes [2][4][8] + K0 shares [8]
  s.rows = off; off += p.ws_rows ? 0 : up(p.R_cap * 4);
  s.red = off; off += up((DEC_MAX_RANKS * 4 + 64) * 4);
  s.chref = off; off += up((DEC_MAX_RANKS + 1) * DEC_WIN * 4);
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

// 64-bit tagged words of the exchange / merge (single-copy atomic when aligned)
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t tag_of(uint64_t v) { return (uint32_t)(v >> 32); }
__device__ __forceinline__ void prefetch_l2_line(const void* g) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(g) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* g, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(g), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

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
  float* partial;          // [splits, B, Hq, d+2]
  int rows_cap;            // rows per smem batch
  int splits;              // CTAs per (b, KV head): CTA s attends to rows [s*cnt/S, (s+1)*cnt/S)
};

}  // namespace hata
