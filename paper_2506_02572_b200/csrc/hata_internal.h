// Internal (non-ABI) declarations shared by the libhata translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

namespace hata {

struct AppendParams {
  const void* k_new;   // [B, Hkv, d] contiguous
  const void* v_new;
  const void* Wh;      // [Hkv, d, rbits]
  void* K;
  void* V;
  int64_t kv_sb, kv_sh, kv_st;
  uint32_t* codes;
  int64_t c_sb, c_sh;
  const int64_t* pos;  // [B] device
  int64_t cap;
  int B, Hkv, d, rbits;
};

struct HashKeysParams {
  const void* K;
  int64_t kv_sb, kv_sh, kv_st;
  const void* Wh;
  uint32_t* codes;
  int64_t c_sb, c_sh;
  int64_t t0, n;       // rows [t0, t0 + n) of every (b, g)
  int64_t cap;         // rows allocated per (b, g) (extent of the TMA tensor map)
  int B, Hkv, d, rbits;
};

cudaError_t launch_append(const AppendParams& p, int is_bf16, cudaStream_t s);
cudaError_t launch_hash_keys_simt(const HashKeysParams& p, int is_bf16, cudaStream_t s);
// tcgen05/TMEM/TMA path (bf16, d == 128, rbits in {32, 64, 128, 256}, K strides
// that one 2-D tensor map covers); cudaErrorNotSupported otherwise.
cudaError_t launch_hash_keys_umma(const HashKeysParams& p, cudaStream_t s);
// fused prefill write (NEXT-1): p.K = K cache, Vdst = V cache, source chunk
// strides ss_*; cudaErrorNotSupported unless 3-D tensor maps cover both sides.
cudaError_t launch_prefill_write_umma(const HashKeysParams& p, const void* Ksrc, const void* Vsrc, int64_t ss_b,
                                      int64_t ss_h, int64_t ss_t, void* Vdst, cudaStream_t s);
// legacy tensor-core path (mma.sync, bf16, d == 128): any strides.
cudaError_t launch_hash_keys_tc(const HashKeysParams& p, cudaStream_t s);

struct DecodePlan {
  int M, stages, chunk, R_cap, rows_cap, nbins, GT, smem;
  bool d_smem, rows_global;
  size_t ws_sync, ws_hist, ws_part, ws_D, ws_rows, ws_total;   // workspace byte offsets / size
};
struct DecodeParams;
// process-wide options (hata_set_option), indices = hata_option values
enum { OPT_SELECTION_HINT = 0, OPT_PDL = 1, OPT_COOPERATIVE = 2, OPT_COUNT = 3 };
int option_value(int opt);
void set_option_value(int opt, int v);
DecodePlan plan_decode(int B, int Hq, int Hkv, int d, int rbits, int64_t n_max, int k, int elem_bytes);
int group_template(int G);
cudaError_t launch_decode(DecodeParams& p, const DecodePlan& plan, void* ws, int is_bf16, cudaStream_t s);

struct SelectParams {
  const int32_t* all_D;    // [P] blocks of [B, Hkv, k], rank_stride elements apart
  const int32_t* all_idx;  // same
  int P, B, Hkv, k, G, rbits;
  int64_t rank_stride;     // elements between consecutive ranks' blocks
  const int64_t* n_total;  // [B]
  int64_t lo, hi;
  int32_t* own_idx;        // [B, Hkv, k]
  int32_t* own_cnt;        // [B, Hkv]
  int32_t* sel_idx;        // [B, Hkv, k] or null
  int32_t* sel_score;      // [B, Hkv, k] or null
};
cudaError_t launch_shard_select(const SelectParams& p, cudaStream_t s);
cudaError_t launch_shard_combine(const float* part, int P, int B, int Hq, int d, void* out, int out_bf16,
                                 cudaStream_t s);
struct PartialParams;
cudaError_t launch_partial_attn(PartialParams& p, int GT, int is_bf16, cudaStream_t s);   // grid: splits x units

int device_sm_count();

}  // namespace hata

namespace hata {
cudaError_t set_decode_trace(void* buf);
}  // namespace hata
namespace hata {
unsigned long long* decode_trace_buf();
}  // namespace hata
namespace hata {
cudaError_t launch_timestamp(void* dst, cudaStream_t s);
}  // namespace hata
