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
//   5  rank-ordered flash-decoding merge of the epoch-tagged partials by
//      min(G, M) merger ranks (one or more heads each)
#pragma once
#include <type_traits>
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

// Two block-wide exclusive scans at once (a and b).  Returns the exclusive
// prefix of a; eb = that of b; ta, tb = the totals.  buf: >= 2 * (DEC_WARPS + 1) ints.
__device__ __forceinline__ int block_excl_scan2(int a, int b, int* buf, int& eb, int& ta, int& tb) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int ia = a, ib = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int ya = __shfl_up_sync(0xffffffffu, ia, o);
    const int yb = __shfl_up_sync(0xffffffffu, ib, o);
    if (lane >= o) { ia += ya; ib += yb; }
  }
  __syncthreads();
  if (lane == 31) { buf[warp] = ia; buf[DEC_WARPS + 1 + warp] = ib; }
  __syncthreads();
  if (warp == 0) {
    const int wa = lane < DEC_WARPS ? buf[lane] : 0, wb = lane < DEC_WARPS ? buf[DEC_WARPS + 1 + lane] : 0;
    int xa = wa, xb = wb;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int ya = __shfl_up_sync(0xffffffffu, xa, o);
      const int yb = __shfl_up_sync(0xffffffffu, xb, o);
      if (lane >= o) { xa += ya; xb += yb; }
    }
    if (lane < DEC_WARPS) { buf[lane] = xa - wa; buf[DEC_WARPS + 1 + lane] = xb - wb; }
    if (lane == DEC_WARPS - 1) { buf[DEC_WARPS] = xa; buf[2 * DEC_WARPS + 1] = xb; }
  }
  __syncthreads();
  ta = buf[DEC_WARPS];
  tb = buf[2 * DEC_WARPS + 1];
  eb = buf[DEC_WARPS + 1 + warp] + ib - b;
  return buf[warp] + ia - a;
}

template <typename T, int W, int GT, int D_HEAD>
__global__ void __launch_bounds__(DEC_THREADS, 1) hata_decode_kernel(const __grid_constant__ DecodeParams p) {
  // signed-weight planes; the G = 5 template uses the odd-G form (two planes
  // of t_b = (G-1)/2 - c_b plus the key's own bits, hata_score.cuh)
  constexpr bool ODDG = GT == 5;
  constexpr int J = ODDG ? 2 : sw_planes_for_group(GT);
  constexpr int STAGE_TOK = DEC_STAGE_BYTES / (W * 4);
  constexpr int EB = sizeof(T);
  constexpr int NSL = AttnState<GT, D_HEAD>::NSL;
  extern __shared__ __align__(1024) uint8_t smem[];
  HATA_TRACE(31);
  HATA_CLK(23);
  if (HATA_DIAG && (p.dbg & 4)) return;                            // diagnostics: launch cost only

  const int M = p.M;
  const bool d_smem = p.d_smem;
  const int cand_mode = p.cand_mode;
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
  uint16_t* Dglob = p.ws_D ? p.ws_D + ((int64_t)u * M + r) * dec_dchunk(p.chunk) : nullptr;
  uint16_t* Dloc = d_smem ? reinterpret_cast<uint16_t*>(smem + L.D) : Dglob;
  uint16_t* Ds = reinterpret_cast<uint16_t*>(smem + L.D);          // Dloc when d_smem (shared-space stores)
  float* qf = reinterpret_cast<float*>(smem + L.qf);
  uint32_t* qw = reinterpret_cast<uint32_t*>(smem + L.qw);
  uint32_t* planes = reinterpret_cast<uint32_t*>(smem + L.planes);   // [2][4][8]
  int32_t* rows = p.ws_rows ? p.ws_rows + ((int64_t)u * M + r) * p.R_cap : reinterpret_cast<int32_t*>(smem + L.rows);
  int32_t* red = reinterpret_cast<int32_t*>(smem + L.red);
  int32_t* misc = reinterpret_cast<int32_t*>(smem + L.misc);
  int32_t* win = reinterpret_cast<int32_t*>(smem + L.chref);       // [M][DEC_WIN] prefix counts near the hint
  int32_t* wtot = win + DEC_MAX_RANKS * DEC_WIN;                    // [DEC_WIN] their unit totals
  float* fmisc = reinterpret_cast<float*>(misc);

  // Rank chunks [rr*per, (rr+1)*per) are fixed by the host from n_max, so the
  // streams start before the device-side length n[b] has arrived.
  const int per = p.chunk;
  const int64_t t0 = (int64_t)r * per;
  const int Lcopy = (int)max((int64_t)0, min((int64_t)per, p.n_max - t0));   // rows streamed
  const int nstages = (Lcopy + STAGE_TOK - 1) / STAGE_TOK;
  const bool recycle = nstages > NST;                              // ring smaller than the chunk
  // row maps of this unit's code cache (words) and K/V caches (elements)
  const int32_t* ptab = p.page_table ? p.page_table + (int64_t)b * p.max_pages : nullptr;
  const RowMap cmap{ptab, p.page_lg, p.c_sb, ptab ? (int64_t)g * p.c_sh : (int64_t)b * p.c_sb + (int64_t)g * p.c_sh,
                    (int64_t)W};
  const RowMap kvmap{ptab, p.page_lg, p.kv_sb,
                     ptab ? (int64_t)g * p.kv_sh : (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh, p.kv_st};
  const T* qg = reinterpret_cast<const T*>(p.q) + ((int64_t)b * p.Hq + (int64_t)g * G) * D_HEAD;
  const bool append = p.k_new != nullptr;
  T* qraw = reinterpret_cast<T*>(smem + L.qraw);                    // [G (+1 key)][d] as stored

  // ---- phase 0: start the q-independent streams with bulk copies (TMA)
  // BEFORE griddepcontrol.wait -- W_g and this rank's code chunk -- so that
  // under programmatic dependent launch they overlap the preceding kernel's
  // tail.  Contract (include/hata.h): a kernel that precedes this launch in
  // the stream and writes code rows makes them visible before it triggers its
  // dependents (every libhata kernel fences, then triggers); the row this
  // launch appends itself is rescored from its own k_new.  q, k_new, v_new,
  // n and the workspace are read after the wait with plain loads (not queued
  // behind the stream's TMA requests).
  // stage s of the code chunk into ring slot s % NST; called by a whole warp
  // (contiguous caches: lane 0 issues one copy; paged: lane i copies the
  // i-th page segment of the stage, the segments' bytes summing to the
  // stage's -- every segment but the chunk's last is a multiple of 16 bytes)
  auto issue_stage = [&](int s) {
    const int slot = s % NST;
    const int ntok = min(STAGE_TOK, Lcopy - s * STAGE_TOK);
    const uint32_t bytes = (uint32_t)(ntok * W * 4) & ~15u;
    const int64_t ts = t0 + (int64_t)s * STAGE_TOK;
    if (lane == 0) mbar_arrive_expect_tx(&bars[slot], bytes);
    __syncwarp();
    if (!ptab) {
      if (lane == 0 && bytes) bulk_g2s(ring + slot * DEC_STAGE_BYTES, p.codes + cmap(ts), bytes, &bars[slot]);
    } else {
      const int ps = 1 << p.page_lg;
      const int64_t first = ts >> p.page_lg, last = (ts + ntok - 1) >> p.page_lg;
      for (int64_t pg = first + lane; ntok > 0 && pg <= last; pg += 32) {
        const int64_t a = max(ts, pg << p.page_lg), z = min(ts + (int64_t)ntok, (pg + 1) << p.page_lg);
        const uint32_t off = (uint32_t)((a - ts) * W * 4);
        const uint32_t nb = min((uint32_t)((z - a) * W * 4), bytes > off ? bytes - off : 0u) & ~15u;
        if (nb) bulk_g2s(ring + slot * DEC_STAGE_BYTES + off, p.codes + cmap(a), nb, &bars[slot]);
      }
      (void)ps;
    }
  };
  const int WROWB = dec_wrow_stride(p.rbits, EB);                   // padded smem row of W_g
  const uint32_t wrow = (uint32_t)(p.rbits * EB);                  // bytes of one W_g row
  if (tid == 0) {
    // [0, NST) code ring, NST: W_g, NST+1: spare, NST+2: spare,
    // NST+3: attention gather batches
    for (int s = 0; s < NST + 4; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&bars[NST], D_HEAD * wrow);
  }
  __syncthreads();                                                  // barriers initialised
  {
    // W_g row by row into padded smem rows (conflict-free ldmatrix), the
    // requests spread over all warps (bulk-copy issue is serial per warp)
    const T* wsrc = reinterpret_cast<const T*>(p.Wh) + (int64_t)g * D_HEAD * p.rbits;
    for (int row = lane * DEC_WARPS + warp; row < D_HEAD; row += DEC_THREADS)
      bulk_g2s(reinterpret_cast<uint8_t*>(Ws) + row * WROWB, wsrc + (int64_t)row * p.rbits, wrow, &bars[NST]);
  }
  __syncthreads();                                                  // W_g requests ahead of the stream
  if (warp == 0 && !ptab)                                           // the code chunk, a few large copies
    for (int s = 0; s < NST && s < nstages; ++s) issue_stage(s);
  for (int i = tid; i < p.nbins; i += DEC_THREADS) hist[i] = 0;
  if (tid < DEC_WIN) wtot[tid] = 0;
  // L2 prefetch of the small inputs read right after the wait (q rows, new
  // key/value rows, n[b], the unit's hint word): a prefetch only moves lines
  // into L2, the point of coherence, so a value the preceding kernel writes
  // is still read after the wait -- it just no longer waits for HBM
  {
    const int qlines = (G * D_HEAD * EB + 127) / 128;
    if (tid < qlines) prefetch_l2_line(reinterpret_cast<const uint8_t*>(qg) + tid * 128);
    else if (append && tid < qlines + 2 * ((D_HEAD * EB + 127) / 128)) {
      const int i = tid - qlines, kl = (D_HEAD * EB + 127) / 128;
      const void* src = i < kl ? p.k_new : p.v_new;
      prefetch_l2_line(reinterpret_cast<const uint8_t*>(src) + (int64_t)u * D_HEAD * EB + (i % kl) * 128);
    } else if (tid == DEC_THREADS - 1) {
      prefetch_l2_line(p.n + b);
      if (p.ws_sync) prefetch_l2_line(p.ws_sync + DEC_SYNC_WORDS * u);
    }
  }
  // Programmatic dependent launch: everything above reads only the hash
  // weights and code rows no preceding kernel writes (contract above); q,
  // k_new, v_new, n, K/V, the workspace and every global write come after
  // the wait.  A no-op without the launch attribute.
  griddep_wait();
  HATA_TRACE(28);
  // n[b] > n_max is clamped to n_max: the rank chunks are fixed by n_max
  // (include/hata.h documents this)
  const int64_t n = min(p.n[b], p.n_max);
  {
    // q rows, then the new key and value rows (16-byte vectors), and the
    // unit's threshold hint of the previous launch
    constexpr int V16 = D_HEAD * EB / 16;                          // 16-byte vectors per row
    const int nv = (G + (append ? 2 : 0)) * V16;
    uint4* dq = reinterpret_cast<uint4*>(qraw);
    for (int i = tid; i < nv; i += DEC_THREADS) {
      const int row = i / V16, c = i % V16;
      const T* src = row < G ? qg + (int64_t)row * D_HEAD
                             : reinterpret_cast<const T*>(row == G ? p.k_new : p.v_new) + (int64_t)u * D_HEAD;
      dq[i] = __ldcg(reinterpret_cast<const uint4*>(src) + c);
    }
    HATA_CLK(17);
    if (tid == DEC_THREADS - 1) {                                    // (not one of the q-row threads)
      // the unit's sync words (two loads in flight): epoch E (this launch
      // tags its exchange and partials with E + 1); the threshold hint of
      // launch E in slot 1 + (E & 1) and the row it appended (+1) in slot
      // 4 + (E & 1) (launch E + 1 writes the other slots)
      const uint4* sp = reinterpret_cast<const uint4*>(p.ws_sync + DEC_SYNC_WORDS * u);
      const uint4 sw = p.ws_sync ? __ldcg(sp) : make_uint4(0, 0, 0, 0);
      const uint4 sw2 = p.ws_sync ? __ldcg(sp + 1) : make_uint4(0, 0, 0, 0);
      // tag E + 1; 0 (the zero-filled workspace) is never a tag: after 2^32
      // launches E + 1 wraps to 2, keeping the epoch parity alternating
      misc[12] = (int)(sw.x + 1u == 0u ? 2u : sw.x + 1u);
      misc[14] = (int)((sw.x & 1u) ? sw.z : sw.y);
      misc[13] = (int)((sw.x & 1u) ? sw2.y : sw2.x);
      HATA_CLK(18);
    }
    if (warp == 0 && ptab)                                          // paged: the page table is read after the wait
      for (int s = 0; s < NST && s < nstages; ++s) issue_stage(s);
  }
  // Candidate hint: the unit's threshold of the previous launch on this
  // workspace (+ DEC_HINT_SLACK).  Tokens with D <= Th are marked in a bitmap
  // while the ranks exchange counts, so that when this launch's threshold is <= Th the
  // selection visits only the marked tokens; otherwise it scans all of D.
  // A hint changes the work done, never the result.
  uint32_t* Bc = reinterpret_cast<uint32_t*>(smem + L.bc);
  const int nbw = d_smem ? dec_dchunk(p.chunk) / 32 : 0;          // bitmap words
  int Th = -1;
  const bool hinted = p.use_hint && p.ws_sync && nbw > 0 && nbw <= DEC_BC_WPT * DEC_THREADS;
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
  const bool owner = append && n >= 1 && pos < p.cap && pos >= t0 && pos < t0 + Lr;
  const int NV = G + (owner ? 1 : 0);                                // projected vectors
  mbar_wait(&bars[NST], 0);                                         // W_g in smem
  __syncthreads();                                                  // q, k_new, v_new, hint in smem
  // previous threshold h: the candidate bitmap marks D <= Th = h + slack; the
  // exchange reads every rank's prefix counts at the window [hw0, hw0 + DEC_WIN)
  int hw0 = 0;
  if (hinted) { const int h = misc[14]; Th = h > 0 ? h + DEC_HINT_SLACK : -1; hw0 = h - (DEC_WIN / 2 - 1); }
  const uint32_t tag = (uint32_t)misc[12];                          // this launch's epoch tag (>= 1)
  const uint64_t tagw = (uint64_t)tag << 32;
  // The row the previous launch on this workspace appended: that launch
  // triggered its dependents without a fence, so this launch's code stream
  // (started before the wait) may hold a stale copy of it -- re-read it now
  // (after the wait) and rescore it after the scoring pass (include/hata.h)
  const int64_t prow = (int64_t)misc[13] - 1;
  const bool reload = prow >= t0 && prow < t0 + Lr && !(append && prow == pos) && prow < p.cap;
  uint32_t* qrel = qw + (GT + 1) * W;                               // its code words
  if (reload && warp == DEC_WARPS - 1 && lane < W) qrel[lane] = __ldcg(p.codes + cmap(prow) + lane);
  HATA_TRACE(9);
  if constexpr (EB != 2) {                                          // fp32 paths read q as floats
    for (int i = tid; i < NV * D_HEAD; i += DEC_THREADS) qf[(i / D_HEAD) * QS + i % D_HEAD] = Elem<T>::to_f(qraw[i]);
    __syncthreads();
  }
  HATA_TRACE(8);
  // signed-weight planes of w_b = G - 2 c_b for code word w (hata_score.cuh):
  // lane = bit of the word, c = #{h: q_h bit set}; P_j / N_j and this word's
  // share of the constant K0 go to smem (whole warp)
  const int sgn_s = (G % 2 == 0) ? 1 : 0;
  auto word_planes = [&](int w, int c) {
    const int v = ODDG ? ((G - 1) >> 1) - c : (G - 2 * c) >> sgn_s;  // exact: G - 2c is even for even G
    const int mag = v < 0 ? -v : v;
    int negc = 0;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const uint32_t pj = __ballot_sync(0xffffffffu, v > 0 && ((mag >> j) & 1));
      const uint32_t nj = __ballot_sync(0xffffffffu, v < 0 && ((mag >> j) & 1));
      negc += __popc(nj) << j;
      if (lane == 0) { planes[j * 8 + w] = pj; planes[32 + j * 8 + w] = nj; }
    }
    const int csum = warp_sum_i(c);
    if (lane == 0) reinterpret_cast<int*>(planes)[64 + w] = csum - (negc << (ODDG ? 1 : sgn_s));   // K0 share of this word
  };
  if constexpr (EB == 2) {
    // bf16: the projection X[NV x d] . W_g[d x rbits] on the tensor cores
    // (mma.sync m16n8k16, exact bf16 products, fp32 accumulation; R13).
    // Warp = one 8-bit column tile of the code; Sign + BitPack (Alg. 2 lines
    // 5-7) straight from the accumulator fragment via ballots.
    const int gid = lane >> 2, tig = lane & 3;
    // A fragments of every k-step, read once from the bf16 rows as stored
    constexpr int KS = D_HEAD / 16;
    uint32_t qa[KS][4];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const uint32_t* x0 = reinterpret_cast<const uint32_t*>(qraw + gid * D_HEAD + ks * 16 + 2 * tig);
      const uint32_t* x1 = reinterpret_cast<const uint32_t*>(qraw + (gid + 8) * D_HEAD + ks * 16 + 2 * tig);
      qa[ks][0] = gid < NV ? x0[0] : 0u;
      qa[ks][1] = gid + 8 < NV ? x1[0] : 0u;
      qa[ks][2] = gid < NV ? x0[4] : 0u;
      qa[ks][3] = gid + 8 < NV ? x1[4] : 0u;
    }
    HATA_CLK(19);
    // warp = one 32-bit code word (4 n-tiles, 4 independent MMA chains);
    // each lane sets its 2 sign bits per n-tile, the 4 lanes of a row OR-reduce
    for (int w = warp; w < W; w += DEC_WARPS) {
      float c[4][4];
#pragma unroll
      for (int q = 0; q < 4; ++q) c[q][0] = c[q][1] = c[q][2] = c[q][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t b0, b1;
          ldsm_x2_trans(b0, b1, reinterpret_cast<const uint8_t*>(Ws) + (ks * 16 + (lane & 15)) * WROWB + (4 * w + q) * 16);
          mma_bf16_16816(c[q], qa[ks], b0, b1);
        }
      HATA_CLK(20);
      uint32_t lo = 0u, hi = 0u;                                    // rows gid / gid + 8, LSB-first (R7)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        lo |= ((uint32_t)(c[q][0] >= 0.f) | ((uint32_t)(c[q][1] >= 0.f) << 1)) << (8 * q + 2 * tig);
        hi |= ((uint32_t)(c[q][2] >= 0.f) | ((uint32_t)(c[q][3] >= 0.f) << 1)) << (8 * q + 2 * tig);
      }
      lo |= __shfl_xor_sync(0xffffffffu, lo, 1);
      hi |= __shfl_xor_sync(0xffffffffu, hi, 1);
      lo |= __shfl_xor_sync(0xffffffffu, lo, 2);
      hi |= __shfl_xor_sync(0xffffffffu, hi, 2);
      if (tig == 0) {
        if (gid < NV) qw[gid * W + w] = lo;
        if (gid + 8 < NV) qw[(gid + 8) * W + w] = hi;
      }
      // the G query words of this code word are in lanes 0, 4, .. (rows = heads
      // < 8): the planes follow in-warp, no smem round trip
      int cnt = 0;
#pragma unroll
      for (int h = 0; h < GT; ++h) {
        const uint32_t wh = __shfl_sync(0xffffffffu, lo, 4 * h);
        if (h < G) cnt += (wh >> lane) & 1u;
      }
      word_planes(w, cnt);
      HATA_CLK(21);
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
  HATA_TRACE(24);
  __syncthreads();
  HATA_TRACE(25);
  // publish the query codes (optional output) and the new key's code (Alg. 3 line 9)
  for (int i = tid; i < NV * W; i += DEC_THREADS) {
    const int h = i / W, w = i % W;
    const uint32_t word = qw[i];
    if (h < G && p.out_qcodes && r == 0) p.out_qcodes[((int64_t)b * p.Hq + g * G + h) * W + w] = word;
    if (h == G) const_cast<uint32_t*>(p.codes)[cmap(pos) + w] = word;
  }
  if constexpr (EB != 2) {                                          // fp32: planes from the smem words
    if (warp < W) {
      int c = 0;
      for (int h = 0; h < G; ++h) c += (qw[h * W + warp] >> lane) & 1u;
      word_planes(warp, c);
    }
    __syncthreads();
  }
  HATA_TRACE(26);
  uint32_t A[J][W], Bp[J][W];                                       // P_j, N_j
#pragma unroll
  for (int j = 0; j < J; ++j)
#pragma unroll
    for (int w = 0; w < W; ++w) { A[j][w] = planes[j * 8 + w]; Bp[j][w] = planes[32 + j * 8 + w]; }
  int K0 = 0;
#pragma unroll
  for (int w = 0; w < W; ++w) K0 += reinterpret_cast<const int*>(planes)[64 + w];
  auto group_D = [&](const uint32_t (&kc)[W]) -> uint32_t {        // D = K0 + (T << s)
    if constexpr (ODDG) return (uint32_t)(K0 + (int)group_distance_odd<W>(kc, A, Bp));
    else return (uint32_t)(K0 + (int)(group_distance_sw<W, J>(kc, A, Bp) << sgn_s));
  };

  HATA_TRACE(1);
  // ---- phase 2: Hamming score + GQA sum (Alg. 3 lines 10-11) + histogram
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
  // one token pair -> one 32-bit store of two u16 distances; SCORE_PAIRS
  // pairs per thread per iteration (independent chains for ILP)
  auto score_pairs = [&](const uint32_t* st, uint32_t* dst, uint32_t* dsts, int npairs) {
#ifndef HATA_SCORE_PAIRS
#define HATA_SCORE_PAIRS 1                                          // measured: 1 beats 2 by ~0.1 us/step (flat loop)
#endif
    constexpr int SP = HATA_SCORE_PAIRS;
    for (int j2 = tid; j2 < npairs; j2 += SP * DEC_THREADS) {
      uint32_t kc[SP][2][W];
      bool ok[SP];
#pragma unroll
      for (int q = 0; q < SP; ++q) {
        const int jq = j2 + q * DEC_THREADS;
        ok[q] = q == 0 || jq < npairs;
        if (ok[q]) { smem_code(st, 2 * jq, kc[q][0]); smem_code(st, 2 * jq + 1, kc[q][1]); }
      }
      uint32_t d[SP][2];
#pragma unroll
      for (int q = 0; q < SP; ++q) { d[q][0] = group_D(kc[q][0]); d[q][1] = group_D(kc[q][1]); }
#pragma unroll
      for (int q = 0; q < SP; ++q) {
        if (!ok[q]) continue;
        if (!(HATA_DIAG && (p.dbg & 2))) {                            // dbg 2: timing without the histogram
          atomicAdd(&hist[d[q][0]], 1u);
          atomicAdd(&hist[d[q][1]], 1u);
        }
        const int jq = j2 + q * DEC_THREADS;
        if (d_smem) dsts[jq] = d[q][0] | (d[q][1] << 16);
        else dst[jq] = d[q][0] | (d[q][1] << 16);
      }
    }
  };
  // leftovers: an odd last token, or tokens past the 16-byte-rounded copy
  auto score_rest = [&](const uint32_t* st, int base, int nval, int copied, int npairs) {
    const int rest = nval - 2 * npairs;
    if (tid < rest) {
      const int j = 2 * npairs + tid;
      uint32_t kc[W];
      if (j < copied) {
        smem_code(st, j, kc);
      } else {
        const uint32_t* gp = p.codes + cmap(t0 + base + j);
#pragma unroll
        for (int w = 0; w < W; ++w) kc[w] = __ldg(gp + w);
      }
      const uint32_t dv = group_D(kc);
      atomicAdd(&hist[dv], 1u);
      Dloc[base + j] = (uint16_t)dv;
    }
  };
  auto copied_tok = [&](int s) {                                   // tokens of stage s fully in smem
    return (int)(((uint32_t)(min(STAGE_TOK, Lcopy - s * STAGE_TOK) * W * 4) & ~15u) / (W * 4));
  };
  if (!recycle) {
    // the whole chunk fits the ring (and was streamed before the wait): one
    // flat pass over it once every stage has landed
    for (int s = 0; s < nstages; ++s) {
      if (!(HATA_DIAG && (p.dbg & 16))) mbar_wait(&bars[s], 0u);
      if (s < 3) HATA_CLK(11 + s);
    }
    HATA_TRACE(10);
    const int copied = nstages ? (nstages - 1) * STAGE_TOK + copied_tok(nstages - 1) : 0;
    const int npairs = max(0, min(Lr, copied)) / 2;
    score_pairs(reinterpret_cast<const uint32_t*>(ring), reinterpret_cast<uint32_t*>(Dloc),
                reinterpret_cast<uint32_t*>(Ds), npairs);
    score_rest(reinterpret_cast<const uint32_t*>(ring), 0, Lr, copied, npairs);
    HATA_TRACE(13);
  } else {
    int slot = 0;
    uint32_t parity = 0;
    for (int s = 0; s < nstages; ++s) {
      if (!(HATA_DIAG && (p.dbg & 16))) mbar_wait(&bars[slot], parity);   // dbg 16: timing without waiting for the stream
      if (s == 0) HATA_TRACE(10);
      if (s == nstages - 1) HATA_TRACE(13);
      const int base = s * STAGE_TOK;
      const int nval = min(STAGE_TOK, Lr - base);                     // valid tokens (< n), may be <= 0
      const int copied = copied_tok(s);
      const int npairs = max(0, min(nval, copied)) / 2;
      const uint32_t* st = reinterpret_cast<const uint32_t*>(ring + slot * DEC_STAGE_BYTES);
      score_pairs(st, reinterpret_cast<uint32_t*>(Dloc + base), reinterpret_cast<uint32_t*>(Ds + base), npairs);
      score_rest(st, base, nval, copied, npairs);
      __syncthreads();                                              // the slot is consumed: refill it
      if (warp == 0 && s + NST < nstages) issue_stage(s + NST);
      if (++slot == NST) { slot = 0; parity ^= 1u; }
    }
  }
  __syncthreads();                                                  // every D / histogram update done
  if (reload && tid == 0) {
    // the previous launch's appended row, re-read after the wait
    uint32_t kc[W];
#pragma unroll
    for (int w = 0; w < W; ++w) kc[w] = qrel[w];
    const int jl = (int)(prow - t0);
    const uint32_t Dn = group_D(kc);
    const uint32_t Do = Dloc[jl];
    hist[Do] -= 1u;
    hist[Dn] += 1u;
    Dloc[jl] = (uint16_t)Dn;
  }
  if (owner && tid == 0) {                                          // (same thread: ordered after the reload)
    // the streamed row pos held the stale code: re-score the appended key
    uint32_t kc[W];
#pragma unroll
    for (int w = 0; w < W; ++w) kc[w] = qw[G * W + w];
    const int jl = (int)(pos - t0);
    const uint32_t Dn = group_D(kc);
    const uint32_t Do = Dloc[jl];
    hist[Do] -= 1u;
    hist[Dn] += 1u;
    Dloc[jl] = (uint16_t)Dn;
  }
  if (owner) {
    // Alg. 3 lines 3-4: K/V rows of the new token (from smem), written before
    // this rank's arrival at the exchange so that every rank's gather sees them
    constexpr int CH = D_HEAD * EB / 16;
    if (tid < 2 * CH) {
      T* dstrow = const_cast<T*>(reinterpret_cast<const T*>(tid < CH ? p.K : p.V)) + kvmap(pos);
      const uint4 v = reinterpret_cast<const uint4*>(qraw + (tid < CH ? G : G + 1) * D_HEAD)[tid % CH];
      reinterpret_cast<uint4*>(dstrow)[tid % CH] = v;
      asm volatile("fence.proxy.async.global;" ::: "memory");        // this rank's own gather reads it by TMA
    }
    // no fence before the trigger: the next launch re-reads this row after
    // its wait (slot 4 + ((E + 1) & 1) records it)
    if (tid == 0 && p.ws_sync) p.ws_sync[DEC_SYNC_WORDS * u + 4 + (tag & 1u)] = (unsigned)(pos + 1);
  }
  // pad D past the valid tokens with 0x7fff (never selected) up to what the
  // selection reads: the per-thread blocking (dec_dchunk(Lr)) of the full
  // scan, or every bitmap word (nbw * 32 = dec_dchunk(chunk)) of the hinted path
  const int dpad = hinted ? nbw * 32 : dec_dchunk(Lr);
  for (int i = Lr + tid; i < dpad; i += DEC_THREADS) Dloc[i] = 0x7fffu;
  __syncthreads();
  // a dependent launch may now start its prologue (W_g + code stream) on the
  // SMs this grid frees; it waits for this grid's completion before reading
  // anything else
  griddep_launch_dependents();

  // ---- phase 3: exact top-k' (Alg. 3 lines 12-13) by counting select.
  // thr = D of the k'-th best token; every D < thr is selected; ties at thr
  // are taken lowest index first (R8): rank by rank (= token order), and in
  // token order inside a rank.  Every rank publishes the exclusive prefix
  // counts of its D histogram (cum_r[i] = #{local D < i}, i = 0..nbins) as
  // epoch-tagged words; each rank polls the M ranks' words (the window
  // around the hint, else every bin) -> the unit totals (-> thr) and the
  // ranks' cum_r[thr], cum_r[thr+1] (-> its tie quota and the output
  // position of its first selected token), then compacts its OWN selected
  // tokens in order and attends to them.
  const int hs = dec_hist_stride(p.nbins + 1);
  HATA_TRACE(2);
  constexpr int BPT_MAX = (8 * 256 + 1 + DEC_THREADS) / DEC_THREADS;  // nbins + 1 <= G*rbits + 2 (G <= 8, rbits <= 256)
  const int BPT = (p.nbins + DEC_THREADS) / DEC_THREADS;
  const int i0 = tid * BPT;
  int tb[BPT_MAX];
  int cum;
  {
    int mysum = 0;
#pragma unroll
    for (int q = 0; q < BPT_MAX; ++q) {
      tb[q] = (q < BPT && i0 + q < p.nbins) ? (int)hist[i0 + q] : 0;
      mysum += tb[q];
    }
    int total;
    // threshold slots, initialised before the scan's barriers (the M == 1
    // threshold loop below writes them without a further barrier)
    if (tid == 0) { misc[0] = -1; misc[1] = 0; misc[4] = p.nbins; }
    cum = block_excl_scan(mysum, misc + 16, total);                  // #{local D < i0}
    HATA_CLK(22);
  }
  auto build_bitmap = [&]() {
    if (Th < 0) return;
    // candidate bitmap (M > 1: while the other ranks arrive): thread t owns
    // words [t*WPT, (t+1)*WPT) (32 tokens each); bit i of word w = (D[32w+i] <= Th)
    const uint32_t th_k = (uint32_t)Th * 0x10001u + 0x80008000u;
    const int WPT = (nbw + DEC_THREADS - 1) / DEC_THREADS;
    // the 16-byte quarters of a word are read in a per-thread rotated order:
    // 8 consecutive threads then touch 8 distinct bank groups (WPT odd)
    const int rot = (WPT & 1) ? (tid >> 1) : tid;
    for (int w = tid * WPT; w < min(nbw, (tid + 1) * WPT); ++w) {
      const uint4* dq = reinterpret_cast<const uint4*>(Dloc + 32 * w);
      uint32_t m = 0u;
#pragma unroll
      for (int c0 = 0; c0 < 4; ++c0) {
        const int c = (c0 + rot) & 3;
        const uint4 x = dq[c];
        const uint32_t a0 = (th_k - x.x) & 0x80008000u, a1 = (th_k - x.y) & 0x80008000u;
        const uint32_t a2 = (th_k - x.z) & 0x80008000u, a3 = (th_k - x.w) & 0x80008000u;
        m |= (((a0 >> 15) & 1u) | ((a0 >> 30) & 2u) | ((a1 >> 13) & 4u) | ((a1 >> 28) & 8u) |
              ((a2 >> 11) & 16u) | ((a2 >> 26) & 32u) | ((a3 >> 9) & 64u) | ((a3 >> 24) & 128u)) << (8 * c);
      }
      Bc[w] = m;
    }
  };
  if (M > 1) {
    // publish this rank's prefix counts as tagged words: no fence and no
    // arrival counter -- a reader that sees this launch's tag sees the count
    uint64_t* gc = p.ws_hist + ((int64_t)u * M + r) * hs;
    const uint64_t* gu = p.ws_hist + (int64_t)u * M * hs;          // rank rr's counts: gu + rr * hs
    int c = cum;
#pragma unroll
    for (int q = 0; q < BPT_MAX; ++q) {
      const int i = i0 + q;
      if (q < BPT && i <= p.nbins) st_relaxed_u64(gc + i, tagw | (uint32_t)c);
      c += tb[q];
    }
    HATA_CLK(24);
    build_bitmap();
    HATA_TRACE(27);
    // the owner's K/V row (generic stores) -> this CTA's gather (async proxy)
    if (tid == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
    // with a hint, every rank's prefix counts at the window bins
    // [w0, w0 + DEC_WIN) around it, polled until each word carries this
    // launch's tag (all of a thread's words in flight at once): the unit
    // totals there give the threshold when it falls in the window, and the
    // per-rank values the tie quota -- one round trip after the last rank
    // publishes
    const int w0 = hw0;
    if (Th >= 0) {
      constexpr int WJ = (DEC_MAX_RANKS * DEC_WIN + DEC_THREADS - 1) / DEC_THREADS;
      uint32_t pend = 0u;
#pragma unroll
      for (int j = 0; j < WJ; ++j) {
        const int i = tid + j * DEC_THREADS, bi = w0 + i % DEC_WIN;
        if (i < M * DEC_WIN) {
          if (bi >= 0 && bi <= p.nbins) pend |= 1u << j;
          else win[i] = 0;
        }
      }
      for (unsigned spins = 0; pend;) {
        uint64_t x[WJ];
#pragma unroll
        for (int j = 0; j < WJ; ++j) {
          const int i = tid + j * DEC_THREADS;
          if ((pend >> j) & 1u) x[j] = ld_relaxed_u64(gu + (int64_t)(i / DEC_WIN) * hs + w0 + i % DEC_WIN);
        }
#pragma unroll
        for (int j = 0; j < WJ; ++j)
          if (((pend >> j) & 1u) && tag_of(x[j]) == tag) {
            win[tid + j * DEC_THREADS] = (int)(uint32_t)x[j];
            atomicAdd(&wtot[(tid + j * DEC_THREADS) % DEC_WIN], (int)(uint32_t)x[j]);
            pend &= ~(1u << j);
          }
        if (pend && ++spins > HATA_SPIN_LIMIT) __trap();           // a lost rank: fail loudly, never hang
      }
    }
    __syncthreads();
    HATA_TRACE(3);
    static_assert(DEC_WIN == 32, "one lane per window bin");
    if (warp == 0) {
      const int tot = Th >= 0 ? wtot[lane] : 0;                       // unit total at bin w0 + lane
      const int z = __shfl_down_sync(0xffffffffu, tot, 1);
      const int bj = w0 + lane;                                       // bins bj, bj + 1 both in the window
      const bool hit = Th >= 0 && lane < DEC_WIN - 1 && bj >= 0 && bj + 1 <= p.nbins && kp > 0 && tot < kp && kp <= z;
      if (hit) { misc[0] = bj; misc[1] = kp - tot; }
      const unsigned any = __ballot_sync(0xffffffffu, hit);
      if (lane == 0) misc[5] = any ? 1 : 0;
    }
    __syncthreads();
    if (!misc[5] && (kp > 0 || r == 0)) {
      // no hint, or the threshold is outside the window: unit totals of
      // every bin from the M ranks' tagged prefix counts -- thread per bin,
      // all M words in flight per poll (one round trip), totals in the code
      // ring (free after scoring), then the crossing bin.  (Rank 0 also
      // runs it when k' = 0: it must have seen every rank's words before it
      // advances the epoch.)
      int32_t* tots = reinterpret_cast<int32_t*>(ring);
      const uint32_t all = M >= 32 ? 0xffffffffu : (1u << M) - 1u;
      for (int j = tid; j <= p.nbins; j += DEC_THREADS) {
        int tot = 0;
        for (uint32_t pend = all, spins = 0; pend;) {
          uint64_t x[DEC_MAX_RANKS];
#pragma unroll
          for (int rr = 0; rr < DEC_MAX_RANKS; ++rr)
            if ((pend >> rr) & 1u) x[rr] = ld_relaxed_u64(gu + (int64_t)rr * hs + j);
#pragma unroll
          for (int rr = 0; rr < DEC_MAX_RANKS; ++rr)
            if (((pend >> rr) & 1u) && tag_of(x[rr]) == tag) { tot += (int)(uint32_t)x[rr]; pend &= ~(1u << rr); }
          if (pend && ++spins > HATA_SPIN_LIMIT) __trap();
        }
        tots[j] = tot;
      }
      __syncthreads();
      for (int j = tid; j < p.nbins; j += DEC_THREADS) {
        const int a = tots[j], z = tots[j + 1];
        if (a < kp && kp <= z) { misc[0] = j; misc[1] = kp - a; }
      }
    }
  } else {
    build_bitmap();
    HATA_TRACE(3);
    int c = cum;
#pragma unroll
    for (int q = 0; q < BPT_MAX; ++q) {
      if (q < BPT && i0 + q < p.nbins && kp > 0 && c < kp && kp <= c + tb[q]) { misc[0] = i0 + q; misc[1] = kp - c; }
      c += tb[q];
    }
  }
  __syncthreads();
  const int thr = misc[0];
  const int need = misc[1];
  if (p.ws_sync && r == 0 && tid == 0) reinterpret_cast<int*>(p.ws_sync)[DEC_SYNC_WORDS * u + 1 + (tag & 1u)] = thr;   // launch E+1's hint slot
  // this rank's tie quota and the selection position of its first token
  // (computed by every warp: no further barrier); the loads are issued here
  // and consumed after the counting pass below
  int quota = need, off0 = 0;
  int bl = 0, ti = 0;
  if (M > 1 && thr >= 0 && lane < M) {
    const int w0 = hw0;                                               // window bins [w0, w0 + DEC_WIN)
    if (Th >= 0 && thr >= w0 && thr + 1 < w0 + DEC_WIN) {
      bl = win[lane * DEC_WIN + thr - w0];
      ti = win[lane * DEC_WIN + thr + 1 - w0];
    } else {
      // outside the window: rank `lane`'s tagged prefix counts at thr, thr + 1
      const uint64_t* cr = p.ws_hist + ((int64_t)u * M + lane) * hs;
      for (unsigned spins = 0;;) {
        const uint64_t x0 = ld_relaxed_u64(cr + thr), x1 = ld_relaxed_u64(cr + thr + 1);
        if (tag_of(x0) == tag && tag_of(x1) == tag) { bl = (int)(uint32_t)x0; ti = (int)(uint32_t)x1; break; }
        if (++spins > HATA_SPIN_LIMIT) __trap();
      }
    }
  }
  HATA_TRACE(11);
  HATA_CLK(0);
  // order-preserving compaction of this rank's selected tokens.  Thread t
  // owns the contiguous tokens [8*S8*t, 8*S8*(t+1)) (the D buffer is padded
  // with 0x7fff to 8*S8*DEC_THREADS, so every load is a full, aligned uint4).
  // Pass 1 counts (D < thr) and (D == thr) per thread with SIMD half-word
  // compares, a warp scan + one barrier give each thread its offsets, pass 2
  // re-reads its tokens and emits the selected ones with predicated,
  // fully unrolled code (no per-token branches, no warp votes).
  int32_t* oidx = p.out_idx ? p.out_idx + (int64_t)u * p.k : nullptr;
  int32_t* osc = p.out_score ? p.out_score + (int64_t)u * p.k : nullptr;
  int32_t* ocd = p.cand_D ? p.cand_D + (int64_t)u * p.k : nullptr;
  const int Gr = G * p.rbits;
  const int S8 = (Lr + 8 * DEC_THREADS - 1) / (8 * DEC_THREADS);   // uint4 (8 tokens) per thread
  const uint4* Dv = reinterpret_cast<const uint4*>(Dloc) + (int64_t)tid * S8;
  // SWAR compares on half-words (every D and the pad 0x7fff are < 2^15):
  // ((x | 0x8000) - d) keeps bit 15 iff d <= x, with no borrow between halves
  const uint32_t lt_k = thr >= 1 ? (uint32_t)(thr - 1) * 0x10001u + 0x80008000u : 0u;   // d <  thr
  const uint32_t le_k = thr >= 0 ? (uint32_t)thr * 0x10001u + 0x80008000u : 0u;         // d <= thr
  // 8-bit mask of a block of 8 tokens from 4 SWAR mask words, bit i = token i
  auto pack8 = [](const uint32_t (&m)[4]) -> uint32_t {
    return ((m[0] >> 15) & 1u) | ((m[0] >> 30) & 2u) | ((m[1] >> 13) & 4u) | ((m[1] >> 28) & 8u) |
           ((m[2] >> 11) & 16u) | ((m[2] >> 26) & 32u) | ((m[3] >> 9) & 64u) | ((m[3] >> 24) & 128u);
  };
  auto swar = [&](uint32_t w, uint32_t& ltw, uint32_t& eqw) {
    ltw = thr >= 1 ? (lt_k - w) & 0x80008000u : 0u;
    const uint32_t lew = thr >= 0 ? (le_k - w) & 0x80008000u : 0u;
    eqw = lew & ~ltw;
  };
  // this rank's tie quota and output offset from the M ranks' prefix counts
  // at thr, thr+1 (lane i: rank i); every warp computes the same values
  auto compute_quota = [&]() {
    if (M > 1 && thr >= 0) {
      ti -= bl;
      int incl = ti;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const int qv = max(0, min(need - (incl - ti), ti));
      const int sel = bl + qv;
      int inc2 = sel;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, inc2, o);
        if (lane >= o) inc2 += v;
      }
      quota = __shfl_sync(0xffffffffu, qv, r);
      off0 = __shfl_sync(0xffffffffu, inc2 - sel, r);
    }
  };
  int Rr = 0;
  // fast path: this launch's threshold is covered by the hint, so every
  // token with D <= thr is marked in Bc; thread t owns the bitmap words
  // [t*WPT, (t+1)*WPT) (token order), visits only the marked tokens, and the
  // picks are emitted in token order from one block scan of the counts
  const bool fast = Th >= 0 && thr >= 0 && thr <= Th;
  if (p.ws_sync && r == 0 && tid == 0) {
    // diagnostics word: launches whose selection took the
    // hinted path (low 16 bits) and whose threshold came from the window
    // exchange (high 16 bits), per unit, wrapping
    unsigned* cnt = p.ws_sync + DEC_SYNC_WORDS * u + 3;
    atomicAdd(cnt, (fast ? 1u : 0u) + ((M > 1 && misc[5]) ? 0x10000u : 0u));   // no return: not on the critical path
  }
  if (fast) {
    const int WPT = (nbw + DEC_THREADS - 1) / DEC_THREADS;
    // WPTC: compile-time bound on the words per thread (1 for chunks of up
    // to 8K tokens, the common multi-rank case; DEC_BC_WPT otherwise)
    auto fast_select = [&](auto wptc) {
      constexpr int WPTC = decltype(wptc)::value;
      uint32_t ltw[WPTC], eqw[WPTC];
      int nlt = 0, neq = 0;
#pragma unroll
      for (int j = 0; j < WPTC; ++j) {
        const int w = tid * WPT + j;
        uint32_t lt = 0u, eq = 0u;
        if (j < WPT && w < nbw && Bc[w]) {
          // the word's 32 distances by SWAR (bounded cost for dense words)
          const uint4* dq = reinterpret_cast<const uint4*>(Dloc + 32 * w);
          const int rot = (WPT & 1) ? (tid >> 1) : tid;               // conflict-free quarter order
#pragma unroll
          for (int c0 = 0; c0 < 4; ++c0) {
            const int c = (c0 + rot) & 3;
            const uint4 x = dq[c];
            uint32_t l4[4], e4[4];
            swar(x.x, l4[0], e4[0]); swar(x.y, l4[1], e4[1]); swar(x.z, l4[2], e4[2]); swar(x.w, l4[3], e4[3]);
            lt |= pack8(l4) << (8 * c);
            eq |= pack8(e4) << (8 * c);
          }
        }
        ltw[j] = lt;
        eqw[j] = eq;
        nlt += __popc(lt);
        neq += __popc(eq);
      }
      HATA_CLK(25);
      int ti_b, lt_tot, ti_tot;
      int lt_b = block_excl_scan2(nlt, neq, misc + 16, ti_b, lt_tot, ti_tot);
      HATA_CLK(26);
      compute_quota();
      HATA_CLK(27);
      Rr = lt_tot + min(ti_tot, quota);
#pragma unroll
      for (int j = 0; j < WPTC; ++j) {
        const int w = tid * WPT + j;
        if (j < WPT && w < nbw && (ltw[j] | eqw[j])) {
          // the first max(0, quota - ti_b) ties of the word are taken (R8)
          uint32_t ties = 0u, e = eqw[j];
          for (int take = min(__popc(e), max(quota - ti_b, 0)); take > 0; --take) {
            ties |= e & (0u - e);
            e &= e - 1u;
          }
          int pl = lt_b + min(ti_b, quota);
          for (uint32_t sel = ltw[j] | ties; sel; sel &= sel - 1u) rows[pl++] = (int32_t)t0 + 32 * w + (__ffs(sel) - 1);
          lt_b += __popc(ltw[j]);
          ti_b += __popc(eqw[j]);
        }
      }
    };
    if (WPT == 1) fast_select(std::integral_constant<int, 1>{});
    else fast_select(std::integral_constant<int, DEC_BC_WPT>{});
  } else {
    int lt_m = 0, eq_m = 0;
    if (thr >= 0) {
      const int rot = tid >> 1;                                       // conflict-free block order (counts only)
  #pragma unroll 4
      for (int c0 = 0; c0 < S8; ++c0) {
        const int c = (c0 + rot) % S8;
        const uint4 x = Dv[c];
        uint32_t l0, e0, l1, e1, l2, e2, l3, e3;
        swar(x.x, l0, e0); swar(x.y, l1, e1); swar(x.z, l2, e2); swar(x.w, l3, e3);
        lt_m += __popc(l0) + __popc(l1) + __popc(l2) + __popc(l3);
        eq_m += __popc(e0) + __popc(e1) + __popc(e2) + __popc(e3);
      }
    }
    HATA_CLK(1);
    // warp-inclusive scans of both counts
    int lt_i = lt_m, eq_i = eq_m;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, lt_i, o), e = __shfl_up_sync(0xffffffffu, eq_i, o);
      if (lane >= o) { lt_i += a; eq_i += e; }
    }
    int* wcnt = misc + 16;                                            // [DEC_WARPS][2] warp totals
    if (lane == 31) { wcnt[2 * warp] = lt_i; wcnt[2 * warp + 1] = eq_i; }
    HATA_CLK(2);
    HATA_TRACE(18);
    compute_quota();
    HATA_CLK(3);
    __syncthreads();
    HATA_CLK(4);
    // this thread's exclusive offsets within the rank, and the rank totals
    int lt_b = lt_i - lt_m, ti_b = eq_i - eq_m, lt_tot = 0, ti_tot = 0;
#pragma unroll
    for (int w = 0; w < DEC_WARPS; ++w) {
      const int cl = wcnt[2 * w], ct = wcnt[2 * w + 1];
      if (w < warp) { lt_b += cl; ti_b += ct; }
      lt_tot += cl;
      ti_tot += ct;
    }
    Rr = lt_tot + min(ti_tot, quota);                                 // rows this rank attends to
    HATA_CLK(5);
    HATA_TRACE(21);
    if (thr >= 0 && lt_m + min(max(quota - ti_b, 0), eq_m) > 0) {
      for (int c = 0; c < S8; ++c) {
        const uint4 x = Dv[c];
        uint32_t lw[4], ew[4];
        swar(x.x, lw[0], ew[0]); swar(x.y, lw[1], ew[1]); swar(x.z, lw[2], ew[2]); swar(x.w, lw[3], ew[3]);
        const uint32_t lt8 = pack8(lw), eq8 = pack8(ew);
        if (lt8 | eq8) {
          // the first max(0, quota - ti_b) ties of the block are taken (R8)
          uint32_t tie8 = 0u, e8 = eq8;
          for (int take = min(__popc(eq8), max(quota - ti_b, 0)); take > 0; --take) {
            tie8 |= e8 & (0u - e8);                                    // lowest remaining tie
            e8 &= e8 - 1u;
          }
          const uint32_t sel8 = lt8 | tie8;
          const int base = lt_b + min(ti_b, quota);                    // position of the block's first pick
          // only the rows list is on the critical path; out_idx / out_score /
          // cand_D are written from it after the attention (coalesced)
          auto emit = [&](int pl, int i) { rows[pl] = (int32_t)t0 + (tid * S8 + c) * 8 + i; };
          if (__popc(sel8) >= 3) {                                     // dense block (e.g. a recent window):
            int rr = 0;                                                // predicated, no per-pick popc
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if ((sel8 >> i) & 1u) emit(base + rr++, i);
          } else {
            for (uint32_t m = sel8; m; m &= m - 1u) {
              const int i = __ffs(m) - 1;
              emit(base + __popc(sel8 & ((1u << i) - 1u)), i);
            }
          }
          lt_b += __popc(lt8);
          ti_b += __popc(eq8);
        }
      }
    }
  }
  HATA_CLK(6);
  HATA_TRACE(22);
#if HATA_DIAG
  if (p.trace && tid == 0) p.trace[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * HATA_TRACE_SLOTS + 32 + 15] = (unsigned long long)Rr;
#endif
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
  if (!cand_mode) {
    const T* Kb = reinterpret_cast<const T*>(p.K) + (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh;
    const T* Vb = reinterpret_cast<const T*>(p.V) + (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh;
    if constexpr (EB == 2) {
      attend_rows_mma<GT, D_HEAD>(rows, Rr, reinterpret_cast<const __nv_bfloat16*>(p.K),
                                  reinterpret_cast<const __nv_bfloat16*>(p.V), kvmap,
                                  reinterpret_cast<const __nv_bfloat16*>(qraw), G, p.scale, smem + L.kv, p.rows_cap, L.rb,
                                  m_s, l_s, st, &bars[NST + 3], &bars[NST + 2],
                                  reinterpret_cast<const uint8_t*>(p.V) == reinterpret_cast<const uint8_t*>(p.K) + D_HEAD * EB &&
                                      p.kv_st == 2 * D_HEAD,
                                  p.trace);
    } else {
      float* sc = reinterpret_cast<float*>(smem + L.sc);
      attend_rows<T, GT, D_HEAD>(rows, Rr, Kb, Vb, p.kv_st, qf, G, p.scale, smem + L.kv, sc, p.rows_cap, L.rb,
                                 m_s, l_s, corr_s, st);
    }
  }
  HATA_TRACE(6);
  // optional outputs of the selection (Alg. 3 line 13): this rank's rows are
  // positions [off0, off0 + Rr) of the ascending k'-list
  if (oidx || osc || ocd) {
    for (int i = tid; i < Rr; i += DEC_THREADS) {
      const int32_t row = rows[i];
      const int dv = (int)Dloc[row - (int32_t)t0];
      if (oidx) oidx[off0 + i] = (int32_t)(row + p.token_offset);
      if (osc) osc[off0 + i] = Gr - 2 * dv;                          // S = G*rbits - 2D
      if (ocd) ocd[off0 + i] = dv;
    }
  }

  // ---- phase 5: merge the M rank partials in rank order (flash-decoding combine)
  const int64_t orow = (int64_t)b * p.Hq + (int64_t)g * G;      // first output row of the group
  auto store_out = [&](int h, int e, float v) {
    const int64_t oi = (orow + h) * D_HEAD + e;
    if (p.out_bf16) reinterpret_cast<__nv_bfloat16*>(p.out)[oi] = __float2bfloat16_rn(v);
    else reinterpret_cast<float*>(p.out)[oi] = v;
  };
  if (M == 1) {
    if (!cand_mode) {
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
    if (p.ws_sync && tid == 0) p.ws_sync[DEC_SYNC_WORDS * u] = tag;              // advance the unit's epoch
    HATA_TRACE(7);
    return;
  }
  // every rank publishes its partial (m, l, acc) as tagged words and is done:
  // no fence, no arrival counter -- ranks >= nmerge exit at once (their SMs
  // go to the next launch); merger rank j < nmerge = min(G, M) polls the
  // words of heads j, j + nmerge, .. until every one carries this launch's
  // tag and merges them in rank order (G mergers: each pulls 1/G of the
  // partial bytes into its SM)
  const int PS = D_HEAD + 2;
  const int PB = dec_part_stride(GT, D_HEAD);
  if (!cand_mode) {
    uint64_t* mypart = p.ws_part + ((int64_t)u * M + r) * PB;
#pragma unroll
    for (int s = 0; s < NSL; ++s) {
      const int sl = tid + s * DEC_THREADS;
      const int h = sl / (D_HEAD / 2), e2 = sl % (D_HEAD / 2);
      if (h < G) {
        st_relaxed_u64(mypart + h * PS + 2 + 2 * e2, tagw | __float_as_uint(st.acc[s][0]));
        st_relaxed_u64(mypart + h * PS + 3 + 2 * e2, tagw | __float_as_uint(st.acc[s][1]));
      }
    }
    if (tid < G) {
      st_relaxed_u64(mypart + tid * PS, tagw | __float_as_uint(m_s[tid]));
      st_relaxed_u64(mypart + tid * PS + 1, tagw | __float_as_uint(l_s[tid]));
    }
  }
  HATA_CLK(8);
  const int nmerge = cand_mode ? 1 : min(G, M);
  if (r >= nmerge) {
    HATA_TRACE(15);
    return;
  }
  HATA_TRACE(15);
  if (!cand_mode) {
    // merger r: heads h = r + nmerge * hi, hi < nh.  The (rank i, head hi)
    // partial rows -- pairs -- are polled warp by warp (warp w: pairs w,
    // w + DEC_WARPS, ..; lane: words lane, lane + 32, .. of the row), every
    // word of a lane in flight per poll, into smem; then warp hi computes
    // the merge weights w[i][hi] = e^{m_i - M_h} and 1 / L_h, and thread
    // (hi, e) sums the M ranks' acc in rank order
    const uint64_t* part = p.ws_part + (int64_t)u * M * PB;
    const int nh = (G - r + nmerge - 1) / nmerge;                     // heads of this merger
    const int npair = M * nh;                                         // <= DEC_MAX_RANKS
    float* pbuf = reinterpret_cast<float*>(smem + L.ring);            // [npair][PS] (the ring is free)
    constexpr int PPW = (DEC_MAX_RANKS + DEC_WARPS - 1) / DEC_WARPS;  // pairs per warp
    constexpr int CPL = (D_HEAD + 2 + 31) / 32;                       // words per lane per pair
    uint32_t pend = 0u;
#pragma unroll
    for (int a = 0; a < PPW; ++a)
#pragma unroll
      for (int c = 0; c < CPL; ++c)
        if (warp + a * DEC_WARPS < npair && lane + 32 * c < PS) pend |= 1u << (a * CPL + c);
    const uint64_t* src[PPW];
#pragma unroll
    for (int a = 0; a < PPW; ++a) {
      const int pr = warp + a * DEC_WARPS, i = pr / nh, hi = pr - i * nh;
      src[a] = part + i * PB + (r + nmerge * hi) * PS + lane;
    }
    for (unsigned spins = 0; pend;) {
      uint64_t x[PPW * CPL];
#pragma unroll
      for (int a = 0; a < PPW; ++a)
#pragma unroll
        for (int c = 0; c < CPL; ++c)
          if ((pend >> (a * CPL + c)) & 1u) x[a * CPL + c] = ld_relaxed_u64(src[a] + 32 * c);
#pragma unroll
      for (int a = 0; a < PPW; ++a)
#pragma unroll
        for (int c = 0; c < CPL; ++c)
          if (((pend >> (a * CPL + c)) & 1u) && tag_of(x[a * CPL + c]) == tag) {
            pbuf[(warp + a * DEC_WARPS) * PS + lane + 32 * c] = __uint_as_float((uint32_t)x[a * CPL + c]);
            pend &= ~(1u << (a * CPL + c));
          }
      if (pend && ++spins > HATA_SPIN_LIMIT) __trap();
    }
    HATA_TRACE(12);
    __syncthreads();
    HATA_TRACE(14);
    // warp = 32 outputs of one head hi: lane i holds rank i's merge weight
    // e^{m_i - M_h} (shuffled into the rank-ordered sum), no smem round trip
    for (int o0 = warp * 32; o0 < nh * D_HEAD; o0 += DEC_THREADS) {
      const int hi = o0 / D_HEAD, e = o0 % D_HEAD + lane;
      const float mr = lane < M ? pbuf[(lane * nh + hi) * PS] : -INFINITY;
      const float lr = lane < M ? pbuf[(lane * nh + hi) * PS + 1] : 0.f;
      float Mx = mr;
#pragma unroll
      for (int x = 16; x > 0; x >>= 1) Mx = fmaxf(Mx, __shfl_xor_sync(0xffffffffu, Mx, x));
      const float w = (mr == -INFINITY) ? 0.f : expf(mr - Mx);
      float Ls = lr * w;
#pragma unroll
      for (int x = 16; x > 0; x >>= 1) Ls += __shfl_xor_sync(0xffffffffu, Ls, x);
      HATA_CLK(29);
      float a0 = 0.f;
#pragma unroll 6
      for (int i = 0; i < M; ++i) a0 = fmaf(pbuf[(i * nh + hi) * PS + 2 + e], __shfl_sync(0xffffffffu, w, i), a0);   // rank order
      store_out(r + nmerge * hi, e, a0 * (Ls > 0.f ? 1.f / Ls : 0.f));
    }
    HATA_CLK(30);
  } else {
    // candidates only: rank 0 has polled every rank's prefix counts (the
    // exchange) before it advances the epoch below
  }
  HATA_CLK(10);
  // advance the unit's epoch: rank 0 has seen a tagged word of every rank
  // (its partials, or in candidates mode the exchange), so every CTA of this
  // launch has read the old epoch
  if (r == 0 && tid == 0) p.ws_sync[DEC_SYNC_WORDS * u] = tag;
  HATA_TRACE(7);
  HATA_CLK(14);
}

}  // namespace hata
