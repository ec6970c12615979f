/*
 * libhata -- C ABI of the B200 (sm_100a) HATA decode hot path.
 *
 * HATA = Hash-Aware Top-k Attention (arXiv 2506.02572).  Citations: "P:n" is
 * line n of the paper text (/root/reference/PAPER.md, LaTeX source), with the
 * algorithm / section it falls in.  Readings R1..R20 of places where the paper
 * is silent are listed in DESIGN.md.
 *
 * CONVENTIONS (all entry points)
 *  - Every pointer is caller-owned DEVICE memory unless stated otherwise; the
 *    library never allocates, frees or synchronises.  HATA-off (P:421-422,
 *    KV offloading): the K and V caches of hata_append / hata_decode_topk_attn
 *    / hata_decode_step may instead be page-locked HOST memory mapped into the
 *    device address space (cudaHostAlloc under UVA); the code cache stays in
 *    device memory, so only the selected K/V rows cross the host link, fetched
 *    by the decode kernel's own gather.  Work is enqueued on
 *    `stream` (a cudaStream_t; NULL = legacy default stream) and is
 *    asynchronous: outputs are valid once the stream reaches that point.
 *  - Argument validation is synchronous and happens before any launch; on a
 *    validation failure nothing is enqueued and outputs are untouched.
 *  - Launch failures return HATA_ERR_CUDA; hata_last_error() has the text.
 *    Faults inside a kernel surface at the caller's next synchronising call.
 *  - Nothing throws across this boundary.
 *  - Tensors:
 *      KV cache   K, V   [B, H_kv, cap, d]  element strides {sb, sh, st},
 *                        d contiguous (stride 1); bf16 or fp32.
 *      code cache codes  [B, H_kv, cap, rbits/32] uint32 word strides
 *                        {sb, sh, st}; st must equal rbits/32 (rows packed),
 *                        rows 16-byte aligned when rbits >= 128.
 *      hash weight W     [H_kv, d, rbits] contiguous, same dtype as K,
 *                        16-byte aligned (one W_H per KV head, shared by its
 *                        G query heads; R4).
 *      queries    q      [B, H_q, d] contiguous, 16-byte aligned; query head h
 *                        reads KV head h / G with G = H_q / H_kv (R5).
 *  - Codes: bit b of a row is 1 iff (x . W[:, b]) >= 0 (sign(0) -> +1, R6),
 *    stored LSB-first in word b / 32 (R7).  Projections accumulate in fp32.
 *  - Supported: d == 128; rbits in {32, 64, 128, 256}; G = H_q/H_kv <= 8;
 *    dtype bf16 or fp32.  Other shapes return HATA_ERR_UNSUPPORTED.
 *  - Thread safety: calls may be made from any host thread; one writer per
 *    cache (the caller orders append before decode on the stream).
 */
#ifndef HATA_H_
#define HATA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HATA_OK = 0,
  HATA_ERR_INVALID_ARG = 1, /* bad shape/pointer/stride (e.g. rbits % 32, H_q % H_kv, k < 1) */
  HATA_ERR_UNSUPPORTED = 2, /* valid but not compiled for this shape/dtype */
  HATA_ERR_CAPACITY = 3,    /* host-checked capacity violation (n > cap) */
  HATA_ERR_WORKSPACE = 4,   /* workspace missing or smaller than hata_decode_workspace_size() */
  HATA_ERR_CUDA = 5         /* a CUDA launch failed; see hata_last_error() */
} hata_status;

typedef enum { HATA_F32 = 0, HATA_BF16 = 1 } hata_dtype;

/* Element (or word) strides of a [B, H_kv, cap, x] tensor; x is contiguous. */
typedef struct {
  int64_t sb, sh, st;
} hata_strides;

typedef struct CUstream_st* hata_stream_t; /* == cudaStream_t */

/* ------------------------------------------------------------------------
 * hata_hash_keys -- HashEncode every cached key of a prefilled cache.
 * PAPER: Alg. 1 "HATA Prefill Stage" lines 2-5 with Alg. 2
 * HashEncode: K_H <- BitPack(Sign(MatMul(K, W_H))); fill the
 * key code cache.
 *   K       [B, H_kv, cap, d] (strides ks), rows [t0, t0 + n) are hashed.
 *   W       [H_kv, d, rbits].
 *   codes   output rows [t0, t0 + n) of [B, H_kv, cap, rbits/32] (strides cs).
 *   cap     rows allocated per (b, KV head) in K and codes; t0 + n > cap ->
 *           CAPACITY (nothing enqueued).
 * bf16 inputs run on the 5th-generation tensor cores: K tiles by TMA
 * (128-byte swizzle), tcgen05.mma with fp32 accumulation in TMEM, W resident
 * in shared memory, tcgen05.ld sign-pack epilogue -- when one 2-D tensor map
 * covers K (its b and h strides are multiples of its row stride), otherwise
 * mma.sync (HMMA); fp32 inputs run on CUDA cores (fp32 FMA).
 * Errors: INVALID_ARG (null pointers, n < 0, rbits % 32, strides),
 *         CAPACITY, UNSUPPORTED (d, rbits, dtype), CUDA.
 * ------------------------------------------------------------------------ */
hata_status hata_hash_keys(const void* K, hata_strides ks, hata_dtype dt, const void* W, int B, int H_kv, int d,
                           int rbits, int64_t t0, int64_t n, int64_t cap, uint32_t* codes, hata_strides cs,
                           hata_stream_t stream);

/* ------------------------------------------------------------------------
 * hata_prefill_write -- write a prefilled chunk into the caches AND hash its
 * keys in one pass (Alg. 1 lines 2-5; the codes
 * come from the K tiles already on chip, so hashing costs no extra HBM read
 * of K -- P:250-251).
 *   K_src, V_src [B, H_kv, n, d] chunk (strides ss; d contiguous).
 *   K, V         caches (strides kvs): rows [t0, t0 + n) of every (b, g) are
 *                written; no other row is touched.
 *   codes        rows [t0, t0 + n) = HashEncode(K_src rows) (strides cs).
 * Both sides must be covered by 3-D tensor maps: batch stride = H_kv x head
 * stride, 16-byte aligned rows.  bf16 only; tcgen05 tensor cores (the
 * hata_hash_keys kernel with a store warp that writes the staged K and V
 * tiles to the caches by TMA).
 * Errors: INVALID_ARG, CAPACITY (t0 + n > cap), UNSUPPORTED (dtype, d, rbits,
 *         strides no 3-D tensor map covers), CUDA.
 * ------------------------------------------------------------------------ */
hata_status hata_prefill_write(const void* K_src, const void* V_src, hata_strides ss, void* K, void* V,
                               hata_strides kvs, hata_dtype dt, const void* W, int B, int H_kv, int d, int rbits,
                               int64_t t0, int64_t n, int64_t cap, uint32_t* codes, hata_strides cs,
                               hata_stream_t stream);

/* ------------------------------------------------------------------------
 * hata_append -- decode-time cache update for the new token.
 * PAPER: Alg. 3 "HATA Decode Stage" lines 2-9: K^cache <- [K^cache; K],
 * V^cache <- [V^cache; V], K_H <- HashEncode(K), K_H^cache <- [K_H^cache; K_H];
 * fused into one kernel as in §4 "Kernel fusion for hash encoding".
 *   k_new, v_new [B, H_kv, d] contiguous, dtype dt.
 *   K, V, codes  caches (strides kvs / cs) written at row pos[b].
 *   pos          DEVICE int64 [B]: row to write (= tokens cached before this step).
 *   cap          rows allocated per (b, g).  A pos[b] outside [0, cap) is skipped
 *                on the device (cannot be validated synchronously).
 * Errors: INVALID_ARG, UNSUPPORTED, CUDA.
 * ------------------------------------------------------------------------ */
hata_status hata_append(const void* k_new, const void* v_new, hata_dtype dt, const void* W, void* K, void* V,
                        hata_strides kvs, uint32_t* codes, hata_strides cs, const int64_t* pos, int64_t cap, int B,
                        int H_kv, int d, int rbits, hata_stream_t stream);

/* ------------------------------------------------------------------------
 * hata_decode_topk_attn -- one decode step over caches that already hold the
 * new token (call hata_append first on the same stream).
 * PAPER: Alg. 3 lines 6 and 10-17, P:254-255:
 *   Q_H  <- HashEncode(q) per query head (W of its KV head, R4/R5);
 *   D[t] <- sum over the G query heads of the group of bitcount(xor(Q_H, K_H^cache[t]))
 *           for t < n[b], including the appended token (R3, R11);
 *   Idx  <- the k' = min(k, n[b]) tokens of smallest D (= largest similarity
 *           S = G*rbits - 2D; R1, R2), ties to the LOWEST index (R8),
 *           reported in ascending order (R9);
 *   out[b, h] <- softmax(scale * q_h . K[Idx]^T) V[Idx]  (Eq. 1, Eq. 2),
 *           gather fused into the attention.
 * Arguments:
 *   q          [B, H_q, d] dtype dt.
 *   K, V       caches (strides kvs), dtype dt.  codes (strides cs).  W as above.
 *   n          DEVICE int64 [B]: tokens per sequence incl. the appended one.
 *   n_max      host upper bound on n[b] (sizes the launch and the workspace);
 *              a device n[b] > n_max is treated as n_max (cannot be validated
 *              synchronously).
 *   k          token budget per (b, KV head), >= 1; k > n[b] clamps (R10).
 *   scale      softmax scale; 0 selects 1/sqrt(d) (R12).
 *   out        [B, H_q, d] dtype out_dt (fp32 recommended for parity, R14).
 *   out_idx    optional [B, H_kv, k] int32: selected token indices ascending,
 *              -1 padding beyond k'.
 *   out_score  optional [B, H_kv, k] int32: S = G*rbits - 2D of those tokens.
 *   out_qcodes optional [B, H_q, rbits/32] uint32: the query codes used.
 *   workspace  device scratch of >= hata_decode_workspace_size(...) bytes,
 *              256-byte aligned, ZERO-FILLED before its first use; one
 *              workspace per concurrently running call.  Per (b, KV head) it
 *              carries 8 words between launches: an epoch (each launch tags
 *              the words its CTAs exchange -- prefix counts, softmax
 *              partials -- with epoch + 1, so readers poll for that tag and
 *              no word is ever reset), and, in two slots chosen by epoch
 *              parity, the last selection threshold and the row the last
 *              fused step appended.  A workspace is tied
 *              to (B, H_kv, G*rbits): launches on it may change n_max and k
 *              (its size must cover the largest), not those three.  It also keeps each
 *              (b, KV head)'s last selection threshold, a hint that lets the
 *              next launch visit only candidate tokens -- it changes the
 *              work, never the result; keep one workspace per attention
 *              layer to keep the hint per layer.  May be NULL when the size
 *              is 0.
 * Launched with programmatic dependent launch (hata_set_option): the kernel
 * streams W and the code rows [0, n_max) into shared memory BEFORE
 * griddepcontrol.wait (they do not depend on q) and reads everything else
 * (q, k_new, v_new, n, K/V, workspace) after it.  Contract: a kernel that
 * precedes this launch in the stream and writes code rows must make those
 * writes visible (__threadfence) before it triggers programmatic completion;
 * hata_hash_keys, hata_prefill_write and hata_append do (fence, then
 * griddepcontrol.launch_dependents), and a kernel that never triggers is
 * complete before this one starts.  The decode kernels themselves trigger
 * without a fence: each records the row it appends in the workspace, and
 * the next decode launch on that workspace re-reads that row after its
 * wait and rescores it (so keep one workspace per cache).  The row a fused
 * decode step appends itself is rescored from its own k_new.
 * One kernel launch of M x (B*H_kv) CTAs (hata_decode_ranks()), at most one
 * per SM; cooperative when HATA_OPT_COOPERATIVE is set.
 * Errors: INVALID_ARG (k < 1, H_q % H_kv, rbits % 32, n_max < 0, nulls),
 *         UNSUPPORTED, WORKSPACE, CUDA.  n[b] == 0 yields zero output and
 *         out_idx all -1.
 * ------------------------------------------------------------------------ */
hata_status hata_decode_topk_attn(const void* q, const void* K, const void* V, hata_strides kvs, hata_dtype dt,
                                  const uint32_t* codes, hata_strides cs, const void* W, int B, int H_q, int H_kv,
                                  int d, int rbits, const int64_t* n, int64_t n_max, int k, float scale, void* out,
                                  hata_dtype out_dt, int32_t* out_idx, int32_t* out_score, uint32_t* out_qcodes,
                                  void* workspace, size_t ws_bytes, hata_stream_t stream);

/* ------------------------------------------------------------------------
 * hata_decode_step -- hata_append + hata_decode_topk_attn in ONE launch:
 * the whole of Alg. 3 (lines 2-17) with the Encode & Cache update
 * fused into the decode kernel (§4 "Kernel fusion for hash encoding").
 *   k_new, v_new [B, H_kv, d] (dtype dt, 16-byte aligned): the new token's key
 *                and value; written with HashEncode(k_new) at row n[b]-1 of
 *                K, V and codes, then scored like every cached token (R11).
 *   n            DEVICE int64 [B]: tokens per sequence INCLUDING the new one.
 *   cap          rows allocated per (b, KV head); n_max > cap -> CAPACITY; a
 *                device row n[b]-1 >= cap is not written.
 * Every other argument as for hata_decode_topk_attn; the result equals
 * hata_append followed by hata_decode_topk_attn.
 * ------------------------------------------------------------------------ */
hata_status hata_decode_step(const void* q, const void* k_new, const void* v_new, void* K, void* V, hata_strides kvs,
                             hata_dtype dt, uint32_t* codes, hata_strides cs, const void* W, int B, int H_q, int H_kv,
                             int d, int rbits, const int64_t* n, int64_t n_max, int64_t cap, int k, float scale,
                             void* out, hata_dtype out_dt, int32_t* out_idx, int32_t* out_score,
                             uint32_t* out_qcodes, void* workspace, size_t ws_bytes, hata_stream_t stream);

/* ------------------------------------------------------------------------
 * hata_decode_step_paged -- hata_decode_step over PAGED caches (the block
 * tables of serving engines; "pluggable into ... FlashInfer/vLLM").
 * Logical token t of sequence b lives in slot t % page_size of physical page
 * page_table[b * max_pages + t / page_size].
 *   K, V   physical pools, element strides kvs = {page stride, head stride,
 *          token stride}, d contiguous (e.g. [pages, H_kv, page_size, 2, d]
 *          with V = K + d: one bulk copy per selected token).
 *   codes  physical pool [pages, H_kv, page_size, rbits/32], word strides
 *          cs = {page stride, head stride, rbits/32}; page and head strides
 *          multiples of 4 words.
 *   page_table  DEVICE int32 [B, max_pages]; entries for pages holding
 *          tokens < n[b] must be valid (the page of row n[b]-1 included: the
 *          step appends there).  The code stream of a paged launch starts
 *          after griddepcontrol.wait (the table may be written by the
 *          preceding kernel).
 *   page_size  a power of two with page_size * rbits/8 a multiple of 16.
 * bf16 only (UNSUPPORTED otherwise); n_max > max_pages * page_size ->
 * CAPACITY; everything else as hata_decode_step.  The prefill hash of a pool
 * is hata_hash_keys over the pool viewed as [pages, H_kv, page_size, d].
 * ------------------------------------------------------------------------ */
hata_status hata_decode_step_paged(const void* q, const void* k_new, const void* v_new, void* K, void* V,
                                   hata_strides kvs, hata_dtype dt, uint32_t* codes, hata_strides cs,
                                   const int32_t* page_table, int max_pages, int page_size, const void* W, int B,
                                   int H_q, int H_kv, int d, int rbits, const int64_t* n, int64_t n_max, int k,
                                   float scale, void* out, hata_dtype out_dt, int32_t* out_idx, int32_t* out_score,
                                   uint32_t* out_qcodes, void* workspace, size_t ws_bytes, hata_stream_t stream);

/* Bytes of device workspace hata_decode_topk_attn needs for this shape
 * (0 when everything fits on chip).  Host-only; never fails (0 on bad args). */
size_t hata_decode_workspace_size(int B, int H_q, int H_kv, int d, int rbits, int64_t n_max, int k,
                                  hata_dtype dt);

/* Number of CTAs ("ranks") per (b, KV head) the decode launch will use, M;
 * the grid is M x (B*H_kv) CTAs.  Host-only; for tests/bench. */
int hata_decode_ranks(int B, int H_q, int H_kv, int d, int rbits, int64_t n_max, int k, hata_dtype dt);

/* ========================================================================
 * Sequence-sharded decode (one rank owns a contiguous token range of every
 * (b, KV head)).  The exchange steps between the
 * phases are the caller's collectives (NCCL all-gather via torch.distributed).
 * Because ranges are contiguous and ascending in rank, "lowest index wins"
 * equals "lower rank first, then local order", so the merged selection is
 * bit-identical to the unsharded one.
 * ======================================================================== */

/* Phase 1: local q-hash + score + local top-k' candidates.
 *   K/V unused here; codes hold this rank's n_local[b] tokens, whose global
 *   index is token_offset + local index.
 *   cand_D    [B, H_kv, k] int32: aggregated distance D of each candidate
 *             (INT32_MAX padding), ascending token order.
 *   cand_idx  [B, H_kv, k] int32: GLOBAL token index (-1 padding).
 * PAPER: Alg. 3 lines 6, 10-13 applied to the rank's slice. */
hata_status hata_shard_candidates(const void* q, hata_dtype dt, const uint32_t* codes, hata_strides cs,
                                  const void* W, int B, int H_q, int H_kv, int d, int rbits, const int64_t* n_local,
                                  int64_t n_local_max, int64_t token_offset, int k, int32_t* cand_D,
                                  int32_t* cand_idx, void* workspace, size_t ws_bytes, hata_stream_t stream);

/* Phase 2: global merge.  all_D / all_idx are the P ranks' candidate lists
 * gathered rank-major: rank r's [B, H_kv, k] block starts rank_stride
 * elements after rank r-1's (0 = B*H_kv*k, i.e. [P, B, H_kv, k]; a packed
 * per-rank [D | idx] buffer gathered with one collective uses 2*B*H_kv*k).
 * Selects the global k' = min(k, n_total[b])
 * smallest (D, index) pairs (identical on every rank) and returns those that
 * fall in [lo, hi) as LOCAL indices (global - lo), ascending, in own_idx
 * [B, H_kv, k] (-1 padding) with counts own_cnt [B, H_kv].  Optionally the
 * whole global selection (ascending) in sel_idx [B, H_kv, k] and its S values
 * in sel_score.  n_total: DEVICE int64 [B]. */
hata_status hata_shard_select(const int32_t* all_D, const int32_t* all_idx, int64_t rank_stride, int P, int B,
                              int H_kv, int k, int G, int rbits, const int64_t* n_total, int64_t lo, int64_t hi,
                              int32_t* own_idx, int32_t* own_cnt, int32_t* sel_idx, int32_t* sel_score,
                              hata_stream_t stream);

/* Phase 3: partial attention over own selected rows, split over `splits`
 * CTAs per (b, KV head) (split s takes rows [s*cnt/S, (s+1)*cnt/S) of the
 * ascending own list; bf16 on the tensor cores, gather fused).
 *   partial [splits, B, H_q, d + 2] fp32: (m, l, acc[d]) with m = max logit
 *   (-inf for an empty split), l = sum exp(z - m), acc = sum exp(z - m) V
 *   (flash-decoding partials; a rank's splits combine like extra ranks). */
hata_status hata_shard_partial_attn(const void* q, const void* K, const void* V, hata_strides kvs, hata_dtype dt,
                                    const int32_t* own_idx, const int32_t* own_cnt, int B, int H_q, int H_kv, int d,
                                    int k, float scale, int splits, float* partial, hata_stream_t stream);

/* Phase 4: combine P partials gathered rank-major [P, B, H_q, d + 2] in rank
 * order (deterministic): M = max m_r, L = sum l_r e^{m_r - M},
 * out = sum acc_r e^{m_r - M} / L. */
hata_status hata_shard_combine(const float* partials, int P, int B, int H_q, int d, void* out, hata_dtype out_dt,
                               hata_stream_t stream);

/* ------------------------------------------------------------------------
 * Process-wide options of the decode launches (defaults: hint 1, PDL 1,
 * cooperative 0).
 *   HATA_OPT_SELECTION_HINT  1: use the previous launch's threshold kept in the
 *                            workspace to visit only candidate tokens in the
 *                            select (changes the work, never the result);
 *                            0: always run the full selection scan.
 *   HATA_OPT_PDL             1: launch with programmatic dependent launch (the
 *                            prologue overlaps the preceding kernel); 0: plain
 *                            stream order.
 *   HATA_OPT_COOPERATIVE     1: decode grids whose ranks exchange (M > 1) are
 *                            cooperative launches (co-residency guaranteed by
 *                            the runtime; a cooperative grid starts only when
 *                            every SM it needs is free, so its prologue cannot
 *                            overlap the preceding kernel); 0: plain launches
 *                            -- the plan never exceeds one CTA per SM, so the
 *                            grid becomes co-resident once the SMs are free,
 *                            but a kernel that holds SMs indefinitely on a
 *                            concurrent stream could stall the ranks' barrier
 *                            (a bounded spin then traps).
 * Returns INVALID_ARG for an unknown option.  Thread safe; affects launches
 * enqueued after the call.
 * ------------------------------------------------------------------------ */
typedef enum { HATA_OPT_SELECTION_HINT = 0, HATA_OPT_PDL = 1, HATA_OPT_COOPERATIVE = 2 } hata_option;
hata_status hata_set_option(hata_option opt, int value);

/* ------------------------------------------------------------------------ */
const char* hata_status_string(hata_status s);
/* Text of the last CUDA error seen by this host thread (empty if none). */
const char* hata_last_error(void);
/* Library version string. */
const char* hata_version(void);

/* Diagnostics only.  buf: NULL (off, the default) or device memory of at least
 * 64 * (number of decode CTAs) uint64; while set, every decode launch writes
 * %globaltimer stamps (ns) of its phase boundaries to buf[cta * 64 + i],
 * i < 32, and clock64 stamps to buf[cta * 64 + 32 + i] (slot meanings:
 * tools/trace_decode.py).  Not for production use. */
hata_status hata_debug_trace(void* buf);
/* Diagnostics only: enqueue a 1-thread kernel that stores %globaltimer (ns)
 * to *dst (device uint64), to bracket a traced launch on the same stream. */
hata_status hata_debug_timestamp(void* dst, hata_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* HATA_H_ */
