// extern "C" boundary of libhata (include/hata.h): synchronous argument
// validation, then one stream-ordered launch per call.  No allocation, no
// synchronisation, no exceptions across the ABI.
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include "../../include/hata.h"
#include "hata_internal.h"
#include "hata_decode.cuh"

namespace {

thread_local char g_last_error[256] = "";

hata_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return HATA_OK;
  std::snprintf(g_last_error, sizeof(g_last_error), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
  return e == cudaErrorNotSupported ? HATA_ERR_UNSUPPORTED : HATA_ERR_CUDA;
}

bool shape_supported(int d, int rbits, int G) {
  return d == 128 && (rbits == 32 || rbits == 64 || rbits == 128 || rbits == 256) && G >= 1 && G <= 8;
}

bool dtype_ok(hata_dtype dt) { return dt == HATA_F32 || dt == HATA_BF16; }

int elem_bytes(hata_dtype dt) { return dt == HATA_BF16 ? 2 : 4; }

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

// Code rows must be packed (st == W) and 16-byte aligned for the bulk copies
// when W >= 4; the per-(b, g) base must be 16-byte aligned too.
bool codes_layout_ok(const void* codes, hata_strides cs, int rbits) {
  const int W = rbits / 32;
  if (cs.st != W) return false;
  const int64_t a = W >= 4 ? 4 : W;  // words
  if (cs.sb % a || cs.sh % a) return false;
  return aligned(codes, (size_t)a * 4);
}

bool kv_layout_ok(const void* K, hata_strides s, int eb, int d) {
  // rows read as d-contiguous vectors of 16 bytes (bf16: 8 elem, f32: 4 elem) per lane group
  const int64_t a = 16 / eb;
  if (s.st < d || s.st % a || s.sh % a || s.sb % a) return false;
  return aligned(K, 16);
}

struct PlanKey {
  int B, Hq, Hkv, d, rbits, k, eb;
  int64_t n_max;
  int dev;
  bool operator<(const PlanKey& o) const {
    return std::tie(B, Hq, Hkv, d, rbits, k, eb, n_max, dev) < std::tie(o.B, o.Hq, o.Hkv, o.d, o.rbits, o.k, o.eb, o.n_max, o.dev);
  }
};
std::mutex g_plan_mu;
std::map<PlanKey, hata::DecodePlan> g_plans;

hata::DecodePlan get_plan(int B, int Hq, int Hkv, int d, int rbits, int64_t n_max, int k, int eb) {
  int dev = -1;
  cudaGetDevice(&dev);
  cudaGetLastError();
  PlanKey key{B, Hq, Hkv, d, rbits, k, eb, n_max, dev};
  {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    auto it = g_plans.find(key);
    if (it != g_plans.end()) return it->second;
  }
  hata::DecodePlan pl = hata::plan_decode(B, Hq, Hkv, d, rbits, n_max, k, eb);
  std::lock_guard<std::mutex> lk(g_plan_mu);
  g_plans[key] = pl;
  return pl;
}

}  // namespace

extern "C" {

const char* hata_status_string(hata_status s) {
  switch (s) {
    case HATA_OK: return "HATA_OK";
    case HATA_ERR_INVALID_ARG: return "HATA_ERR_INVALID_ARG";
    case HATA_ERR_UNSUPPORTED: return "HATA_ERR_UNSUPPORTED";
    case HATA_ERR_CAPACITY: return "HATA_ERR_CAPACITY";
    case HATA_ERR_WORKSPACE: return "HATA_ERR_WORKSPACE";
    case HATA_ERR_CUDA: return "HATA_ERR_CUDA";
  }
  return "HATA_ERR_UNKNOWN";
}

const char* hata_last_error(void) { return g_last_error; }

hata_status hata_set_option(hata_option opt, int value) {
  if (opt != HATA_OPT_SELECTION_HINT && opt != HATA_OPT_PDL && opt != HATA_OPT_COOPERATIVE) return HATA_ERR_INVALID_ARG;
  hata::set_option_value((int)opt, value ? 1 : 0);
  return HATA_OK;
}

const char* hata_version(void) { return "libhata 0.1 (sm_100a)"; }

hata_status hata_debug_trace(void* buf) { return cuda_status(hata::set_decode_trace(buf)); }

hata_status hata_debug_timestamp(void* dst, hata_stream_t stream) {
  if (!dst) return HATA_ERR_INVALID_ARG;
  return cuda_status(hata::launch_timestamp(dst, reinterpret_cast<cudaStream_t>(stream)));
}

hata_status hata_hash_keys(const void* K, hata_strides ks, hata_dtype dt, const void* W, int B, int H_kv, int d,
                           int rbits, int64_t t0, int64_t n, int64_t cap, uint32_t* codes, hata_strides cs,
                           hata_stream_t stream) {
  if (!K || !W || !codes || B < 1 || H_kv < 1 || d < 1 || rbits < 32 || rbits % 32 || t0 < 0 || n < 0 ||
      !dtype_ok(dt))
    return HATA_ERR_INVALID_ARG;
  if (t0 + n > cap) return HATA_ERR_CAPACITY;
  if (!shape_supported(d, rbits, 1)) return HATA_ERR_UNSUPPORTED;
  if (!kv_layout_ok(K, ks, elem_bytes(dt), d) || cs.st != rbits / 32 || !aligned(codes, 4) || !aligned(W, 16))
    return HATA_ERR_INVALID_ARG;
  if (n == 0) return HATA_OK;
  hata::HashKeysParams p = {};
  p.K = K; p.kv_sb = ks.sb; p.kv_sh = ks.sh; p.kv_st = ks.st;
  p.Wh = W; p.codes = codes; p.c_sb = cs.sb; p.c_sh = cs.sh;
  p.t0 = t0; p.n = n; p.cap = cap; p.B = B; p.Hkv = H_kv; p.d = d; p.rbits = rbits;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (dt == HATA_BF16) {
    cudaError_t e = hata::launch_hash_keys_umma(p, s);         // tcgen05 + TMEM + TMA
    if (e != cudaErrorNotSupported) return cuda_status(e);
    e = hata::launch_hash_keys_tc(p, s);                       // strides no tensor map covers: mma.sync
    if (e != cudaErrorNotSupported) return cuda_status(e);
  }
  return cuda_status(hata::launch_hash_keys_simt(p, dt == HATA_BF16, s));
}

hata_status hata_prefill_write(const void* K_src, const void* V_src, hata_strides ss, void* K, void* V,
                               hata_strides kvs, hata_dtype dt, const void* W, int B, int H_kv, int d, int rbits,
                               int64_t t0, int64_t n, int64_t cap, uint32_t* codes, hata_strides cs,
                               hata_stream_t stream) {
  if (!K_src || !V_src || !K || !V || !W || !codes || B < 1 || H_kv < 1 || rbits < 32 || rbits % 32 || t0 < 0 ||
      n < 0 || !dtype_ok(dt))
    return HATA_ERR_INVALID_ARG;
  if (t0 + n > cap) return HATA_ERR_CAPACITY;
  if (!shape_supported(d, rbits, 1) || dt != HATA_BF16) return HATA_ERR_UNSUPPORTED;
  if (!kv_layout_ok(K, kvs, 2, d) || !kv_layout_ok(V, kvs, 2, d) || !kv_layout_ok(K_src, ss, 2, d) ||
      !kv_layout_ok(V_src, ss, 2, d) || cs.st != rbits / 32 || !aligned(codes, 4) || !aligned(W, 16))
    return HATA_ERR_INVALID_ARG;
  if (n == 0) return HATA_OK;
  hata::HashKeysParams p = {};
  p.K = K; p.kv_sb = kvs.sb; p.kv_sh = kvs.sh; p.kv_st = kvs.st;
  p.Wh = W; p.codes = codes; p.c_sb = cs.sb; p.c_sh = cs.sh;
  p.t0 = t0; p.n = n; p.cap = cap; p.B = B; p.Hkv = H_kv; p.d = d; p.rbits = rbits;
  return cuda_status(hata::launch_prefill_write_umma(p, K_src, V_src, ss.sb, ss.sh, ss.st, V,
                                                     reinterpret_cast<cudaStream_t>(stream)));
}

hata_status hata_append(const void* k_new, const void* v_new, hata_dtype dt, const void* W, void* K, void* V,
                        hata_strides kvs, uint32_t* codes, hata_strides cs, const int64_t* pos, int64_t cap, int B,
                        int H_kv, int d, int rbits, hata_stream_t stream) {
  if (!k_new || !v_new || !W || !K || !V || !codes || !pos || cap < 1 || B < 1 || H_kv < 1 || rbits < 32 ||
      rbits % 32 || !dtype_ok(dt))
    return HATA_ERR_INVALID_ARG;
  if (!shape_supported(d, rbits, 1)) return HATA_ERR_UNSUPPORTED;
  if (!kv_layout_ok(K, kvs, elem_bytes(dt), d) || !kv_layout_ok(V, kvs, elem_bytes(dt), d) || cs.st != rbits / 32)
    return HATA_ERR_INVALID_ARG;
  hata::AppendParams p = {};
  p.k_new = k_new; p.v_new = v_new; p.Wh = W; p.K = K; p.V = V;
  p.kv_sb = kvs.sb; p.kv_sh = kvs.sh; p.kv_st = kvs.st;
  p.codes = codes; p.c_sb = cs.sb; p.c_sh = cs.sh; p.pos = pos; p.cap = cap;
  p.B = B; p.Hkv = H_kv; p.d = d; p.rbits = rbits;
  return cuda_status(hata::launch_append(p, dt == HATA_BF16, reinterpret_cast<cudaStream_t>(stream)));
}

size_t hata_decode_workspace_size(int B, int H_q, int H_kv, int d, int rbits, int64_t n_max, int k, hata_dtype dt) {
  if (B < 1 || H_kv < 1 || H_q < H_kv || H_q % H_kv || rbits % 32 || n_max < 0 || k < 1 || !dtype_ok(dt)) return 0;
  if (!shape_supported(d, rbits, H_q / H_kv)) return 0;
  return get_plan(B, H_q, H_kv, d, rbits, n_max, k, elem_bytes(dt)).ws_total;
}

int hata_decode_ranks(int B, int H_q, int H_kv, int d, int rbits, int64_t n_max, int k, hata_dtype dt) {
  if (B < 1 || H_kv < 1 || H_q < H_kv || H_q % H_kv || rbits % 32 || n_max < 0 || k < 1 || !dtype_ok(dt)) return 0;
  if (!shape_supported(d, rbits, H_q / H_kv)) return 0;
  return get_plan(B, H_q, H_kv, d, rbits, n_max, k, elem_bytes(dt)).M;
}

static hata_status decode_common(const void* q, const void* K, const void* V, hata_strides kvs, hata_dtype dt,
                                 const uint32_t* codes, hata_strides cs, const void* W, int B, int H_q, int H_kv,
                                 int d, int rbits, const int64_t* n, int64_t n_max, int k, float scale, void* out,
                                 hata_dtype out_dt, int32_t* out_idx, int32_t* out_score, uint32_t* out_qcodes,
                                 void* workspace, size_t ws_bytes, int cand_mode, int64_t token_offset,
                                 int32_t* cand_D, const void* k_new, const void* v_new, int64_t cap,
                                 hata_stream_t stream, const int32_t* page_table = nullptr, int max_pages = 0,
                                 int page_lg = 0) {
  if (!q || !codes || !W || !n || B < 1 || H_kv < 1 || H_q < H_kv || H_q % H_kv || rbits < 32 || rbits % 32 ||
      n_max < 0 || k < 1 || !dtype_ok(dt))
    return HATA_ERR_INVALID_ARG;
  if (!cand_mode && (!K || !V || !out || !dtype_ok(out_dt))) return HATA_ERR_INVALID_ARG;
  if (!shape_supported(d, rbits, H_q / H_kv)) return HATA_ERR_UNSUPPORTED;
  if (n_max > INT32_MAX / 2) return HATA_ERR_UNSUPPORTED;
  if (!codes_layout_ok(codes, cs, rbits)) return HATA_ERR_INVALID_ARG;
  if (!cand_mode && (!kv_layout_ok(K, kvs, elem_bytes(dt), d) || !kv_layout_ok(V, kvs, elem_bytes(dt), d)))
    return HATA_ERR_INVALID_ARG;
  if (!aligned(q, 16) || !aligned(W, 16)) return HATA_ERR_INVALID_ARG;   // bulk-copied (TMA)
  const hata::DecodePlan pl = get_plan(B, H_q, H_kv, d, rbits, n_max, k, elem_bytes(dt));
  if (pl.GT < 0) return HATA_ERR_UNSUPPORTED;
  if (pl.ws_total && (!workspace || ws_bytes < pl.ws_total || !aligned(workspace, 256))) return HATA_ERR_WORKSPACE;
  hata::DecodeParams p = {};
  p.q = q; p.K = K; p.V = V; p.kv_sb = kvs.sb; p.kv_sh = kvs.sh; p.kv_st = kvs.st;
  p.codes = codes; p.c_sb = cs.sb; p.c_sh = cs.sh; p.Wh = W; p.n = n;
  p.B = B; p.Hq = H_q; p.Hkv = H_kv; p.G = H_q / H_kv; p.d = d; p.rbits = rbits; p.k = k; p.n_max = n_max;
  p.scale = scale != 0.f ? scale : 1.0f / sqrtf((float)d);
  p.out = out; p.out_bf16 = out_dt == HATA_BF16;
  p.out_idx = out_idx; p.out_score = out_score; p.out_qcodes = out_qcodes;
  p.cand_mode = cand_mode; p.token_offset = token_offset; p.cand_D = cand_D;
  p.k_new = k_new; p.v_new = v_new; p.cap = cap;
  p.page_table = page_table; p.max_pages = max_pages; p.page_lg = page_lg;
  return cuda_status(hata::launch_decode(p, pl, workspace, dt == HATA_BF16, reinterpret_cast<cudaStream_t>(stream)));
}

hata_status hata_decode_topk_attn(const void* q, const void* K, const void* V, hata_strides kvs, hata_dtype dt,
                                  const uint32_t* codes, hata_strides cs, const void* W, int B, int H_q, int H_kv,
                                  int d, int rbits, const int64_t* n, int64_t n_max, int k, float scale, void* out,
                                  hata_dtype out_dt, int32_t* out_idx, int32_t* out_score, uint32_t* out_qcodes,
                                  void* workspace, size_t ws_bytes, hata_stream_t stream) {
  return decode_common(q, K, V, kvs, dt, codes, cs, W, B, H_q, H_kv, d, rbits, n, n_max, k, scale, out, out_dt,
                       out_idx, out_score, out_qcodes, workspace, ws_bytes, 0, 0, nullptr, nullptr, nullptr, n_max, stream);
}

hata_status hata_decode_step(const void* q, const void* k_new, const void* v_new, void* K, void* V, hata_strides kvs,
                             hata_dtype dt, uint32_t* codes, hata_strides cs, const void* W, int B, int H_q, int H_kv,
                             int d, int rbits, const int64_t* n, int64_t n_max, int64_t cap, int k, float scale,
                             void* out, hata_dtype out_dt, int32_t* out_idx, int32_t* out_score,
                             uint32_t* out_qcodes, void* workspace, size_t ws_bytes, hata_stream_t stream) {
  if (!k_new || !v_new) return HATA_ERR_INVALID_ARG;
  if (n_max > cap) return HATA_ERR_CAPACITY;
  if (!aligned(k_new, 16) || !aligned(v_new, 16)) return HATA_ERR_INVALID_ARG;
  return decode_common(q, K, V, kvs, dt, codes, cs, W, B, H_q, H_kv, d, rbits, n, n_max, k, scale, out, out_dt,
                       out_idx, out_score, out_qcodes, workspace, ws_bytes, 0, 0, nullptr, k_new, v_new, cap, stream);
}

hata_status hata_decode_step_paged(const void* q, const void* k_new, const void* v_new, void* K, void* V,
                                   hata_strides kvs, hata_dtype dt, uint32_t* codes, hata_strides cs,
                                   const int32_t* page_table, int max_pages, int page_size, const void* W, int B,
                                   int H_q, int H_kv, int d, int rbits, const int64_t* n, int64_t n_max, int k,
                                   float scale, void* out, hata_dtype out_dt, int32_t* out_idx, int32_t* out_score,
                                   uint32_t* out_qcodes, void* workspace, size_t ws_bytes, hata_stream_t stream) {
  if (!k_new || !v_new || !page_table || max_pages < 1 || page_size < 1) return HATA_ERR_INVALID_ARG;
  int lg = 0;
  while ((1 << lg) < page_size) ++lg;
  if ((1 << lg) != page_size) return HATA_ERR_INVALID_ARG;                  // a power of two
  if (dt != HATA_BF16) return HATA_ERR_UNSUPPORTED;
  if (((int64_t)page_size * (rbits / 32) * 4) % 16 || cs.sb % 4 || cs.sh % 4) return HATA_ERR_INVALID_ARG;
  if (n_max > (int64_t)max_pages * page_size) return HATA_ERR_CAPACITY;
  if (!aligned(k_new, 16) || !aligned(v_new, 16)) return HATA_ERR_INVALID_ARG;
  // kvs / cs: {page stride, head stride, token stride}; a sequence's capacity is max_pages pages
  return decode_common(q, K, V, kvs, dt, codes, cs, W, B, H_q, H_kv, d, rbits, n, n_max, k, scale, out, out_dt,
                       out_idx, out_score, out_qcodes, workspace, ws_bytes, 0, 0, nullptr, k_new, v_new,
                       (int64_t)max_pages * page_size, stream, page_table, max_pages, lg);
}

hata_status hata_shard_candidates(const void* q, hata_dtype dt, const uint32_t* codes, hata_strides cs,
                                  const void* W, int B, int H_q, int H_kv, int d, int rbits, const int64_t* n_local,
                                  int64_t n_local_max, int64_t token_offset, int k, int32_t* cand_D,
                                  int32_t* cand_idx, void* workspace, size_t ws_bytes, hata_stream_t stream) {
  if (!cand_D || !cand_idx || token_offset < 0 || token_offset + n_local_max > INT32_MAX)
    return HATA_ERR_INVALID_ARG;
  hata_strides none = {0, 0, 0};
  return decode_common(q, nullptr, nullptr, none, dt, codes, cs, W, B, H_q, H_kv, d, rbits, n_local, n_local_max, k,
                       0.f, nullptr, HATA_F32, cand_idx, nullptr, nullptr, workspace, ws_bytes, 1, token_offset,
                       cand_D, nullptr, nullptr, n_local_max, stream);
}

hata_status hata_shard_select(const int32_t* all_D, const int32_t* all_idx, int64_t rank_stride, int P, int B,
                              int H_kv, int k, int G, int rbits, const int64_t* n_total, int64_t lo, int64_t hi,
                              int32_t* own_idx, int32_t* own_cnt, int32_t* sel_idx, int32_t* sel_score,
                              hata_stream_t stream) {
  if (!all_D || !all_idx || !n_total || !own_idx || !own_cnt || P < 1 || B < 1 || H_kv < 1 || k < 1 || G < 1 ||
      rbits % 32 || lo < 0 || hi < lo || rank_stride < 0)
    return HATA_ERR_INVALID_ARG;
  if (rank_stride == 0) rank_stride = (int64_t)B * H_kv * k;
  if (rank_stride < (int64_t)B * H_kv * k) return HATA_ERR_INVALID_ARG;
  if ((size_t)(G * rbits + 1 + k + 64) * 4 > 200 * 1024) return HATA_ERR_UNSUPPORTED;
  hata::SelectParams p = {all_D, all_idx, P, B, H_kv, k, G, rbits, rank_stride, n_total, lo, hi, own_idx, own_cnt,
                          sel_idx, sel_score};
  return cuda_status(hata::launch_shard_select(p, reinterpret_cast<cudaStream_t>(stream)));
}

hata_status hata_shard_partial_attn(const void* q, const void* K, const void* V, hata_strides kvs, hata_dtype dt,
                                    const int32_t* own_idx, const int32_t* own_cnt, int B, int H_q, int H_kv, int d,
                                    int k, float scale, int splits, float* partial, hata_stream_t stream) {
  if (!q || !K || !V || !own_idx || !own_cnt || !partial || B < 1 || H_kv < 1 || H_q % H_kv || k < 1 ||
      splits < 1 || !dtype_ok(dt))
    return HATA_ERR_INVALID_ARG;
  if (!shape_supported(d, 128, H_q / H_kv)) return HATA_ERR_UNSUPPORTED;
  if (!kv_layout_ok(K, kvs, elem_bytes(dt), d) || !kv_layout_ok(V, kvs, elem_bytes(dt), d)) return HATA_ERR_INVALID_ARG;
  hata::PartialParams p = {};
  p.q = q; p.K = K; p.V = V; p.kv_sb = kvs.sb; p.kv_sh = kvs.sh; p.kv_st = kvs.st;
  p.own_idx = own_idx; p.own_cnt = own_cnt;
  p.B = B; p.Hq = H_q; p.Hkv = H_kv; p.G = H_q / H_kv; p.d = d; p.k = k;
  p.scale = scale != 0.f ? scale : 1.0f / sqrtf((float)d);
  p.partial = partial;
  p.splits = splits;
  const int G = H_q / H_kv;
  const int GT = hata::group_template(G);
  return cuda_status(hata::launch_partial_attn(p, GT, dt == HATA_BF16, reinterpret_cast<cudaStream_t>(stream)));
}

hata_status hata_shard_combine(const float* partials, int P, int B, int H_q, int d, void* out, hata_dtype out_dt,
                               hata_stream_t stream) {
  if (!partials || !out || P < 1 || B < 1 || H_q < 1 || d < 1 || !dtype_ok(out_dt)) return HATA_ERR_INVALID_ARG;
  return cuda_status(
      hata::launch_shard_combine(partials, P, B, H_q, d, out, out_dt == HATA_BF16, reinterpret_cast<cudaStream_t>(stream)));
}

}  // extern "C"
