// Host-side planning + dispatch of the fused decode kernel (hata_decode.cuh).
#include <atomic>
#include <cstdlib>
#include "hata_internal.h"
#include "hata_decode_kernel.cuh"

namespace hata {

constexpr int SMEM_LIMIT = 227 * 1024;
constexpr int ROWS_SMEM_MAX = 4096;            // selected rows per rank kept in smem

int device_sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) n = 148;
  }
  cudaGetLastError();
  return n;
}

int group_template(int G) {
  if (G <= 1) return 1;
  if (G <= 2) return 2;
  if (G <= 4) return 4;
  if (G <= 5) return 5;
  if (G <= 8) return 8;
  return -1;
}

typedef void (*DecodeKernel)(const DecodeParams);

#if !HATA_ONLY_HOT
template <typename T, int W>
static DecodeKernel pick_gt(int GT) {
  switch (GT) {
    case 1: return hata_decode_kernel<T, W, 1, 128>;
    case 2: return hata_decode_kernel<T, W, 2, 128>;
    case 4: return hata_decode_kernel<T, W, 4, 128>;
    case 5: return hata_decode_kernel<T, W, 5, 128>;
    case 8: return hata_decode_kernel<T, W, 8, 128>;
  }
  return nullptr;
}
template <typename T>
static DecodeKernel pick_w(int W, int GT) {
  switch (W) {
    case 1: return pick_gt<T, 1>(GT);
    case 2: return pick_gt<T, 2>(GT);
    case 4: return pick_gt<T, 4>(GT);
    case 8: return pick_gt<T, 8>(GT);
  }
  return nullptr;
}
#endif
static DecodeKernel get_kernel(int is_bf16, int W, int GT) {
#if HATA_ONLY_HOT
  // experimental builds (HATA_DEFS=-DHATA_ONLY_HOT=1): only the bf16,
  // rbits = 128, G = 4 instantiation (the CFG-2/3/4 shape), for fast A/B builds
  return (is_bf16 && W == 4 && GT == 4) ? hata_decode_kernel<__nv_bfloat16, 4, 4, 128> : nullptr;
#else
  return is_bf16 ? pick_w<__nv_bfloat16>(W, GT) : pick_w<float>(W, GT);
#endif
}

static size_t up256(size_t x) { return (x + 255) / 256 * 256; }

// Decomposition + shared-memory + workspace plan (pure function of the shape
// and the device's SM count; cached by the ABI layer).
DecodePlan plan_decode(int B, int Hq, int Hkv, int d, int rbits, int64_t n_max, int k, int eb) {
  DecodePlan pl = {};
  const int G = Hq / Hkv;
  pl.GT = group_template(G);
  pl.nbins = G * rbits + 1;
  const int GT = pl.GT > 0 ? pl.GT : 1;
  const int units = B * Hkv;
  const int sms = device_sm_count();
  int M = sms / (units > 0 ? units : 1);
  if (M < 1) M = 1;
  if (M > DEC_MAX_RANKS) M = DEC_MAX_RANKS;
  const int64_t by_len = (n_max + 1023) / 1024;          // >= 1024 tokens per rank
  if (by_len < M) M = (int)(by_len < 1 ? 1 : by_len);
#if HATA_DIAG
  // diagnostics build only: force the rank count
  if (const char* e = std::getenv("HATA_RANKS")) {
    const int v = std::atoi(e);
    if (v >= 1 && v <= DEC_MAX_RANKS && v * units <= sms) M = v;
  }
#endif
  const int rowb = d * eb + DEC_ROW_PAD;
  const int wbytes = (d * dec_wrow_stride(rbits, eb) + 127) & ~127;
  for (;;) {
    pl.M = M;
    const int64_t per = (n_max + M - 1) / M;
    pl.chunk = (int)((per + DEC_CHUNK_ALIGN - 1) / DEC_CHUNK_ALIGN * DEC_CHUNK_ALIGN);
    if (pl.chunk < DEC_CHUNK_ALIGN) pl.chunk = DEC_CHUNK_ALIGN;
    const int64_t kmax = k < n_max ? k : n_max;
    pl.R_cap = (int)(kmax < pl.chunk ? kmax : pl.chunk);         // a rank may hold every selected row
    if (pl.R_cap < 1) pl.R_cap = 1;
    pl.rows_global = pl.R_cap > ROWS_SMEM_MAX;
    // shared memory: the code ring holds the whole chunk when it can (8 x 16 KB);
    // prefer keeping D on chip over a deep ring (shrink to 4 stages first)
    DecodeParams sp = {};
    sp.d = d; sp.rbits = rbits; sp.nbins = pl.nbins; sp.chunk = pl.chunk; sp.rows_cap = 1;
    sp.R_cap = pl.R_cap; sp.ws_rows = pl.rows_global ? reinterpret_cast<int32_t*>(256) : nullptr;
    sp.d_smem = 1;
    pl.stages = DEC_MAX_STAGES;
    for (;; --pl.stages) {
      sp.stages = pl.stages;
      pl.smem = decode_smem_layout(sp, GT, eb).total;
      if (pl.smem <= SMEM_LIMIT || pl.stages == 2) break;
    }
    pl.d_smem = pl.smem <= SMEM_LIMIT;
    if (!pl.d_smem) {
      sp.d_smem = 0;
      pl.stages = DEC_MAX_STAGES;
      for (;; --pl.stages) {
        sp.stages = pl.stages;
        pl.smem = decode_smem_layout(sp, GT, eb).total;
        if (pl.smem <= SMEM_LIMIT || pl.stages == 2) break;
      }
    }
    // the ring + W area is reused after scoring: histograms of all ranks, the
    // staged K/V rows of one attention batch, the partials of all ranks
    const int region = pl.stages * DEC_STAGE_BYTES + wbytes;
    int rc = region / (2 * rowb + GT * 4) - 1;
    if (rc > pl.R_cap) rc = pl.R_cap;
    if (rc < 1) rc = 1;
    pl.rows_cap = rc;
    break;
  }
  const int hs = dec_hist_stride(pl.nbins + 1);
  // workspace (every section 256-byte aligned).  The one section that
  // carries state from one launch to the next -- the sync words (zero
  // between launches, plus the threshold hint) -- comes first, at an offset
  // that does not depend on the shape, so a workspace may be reused while
  // n_max (hence M) and k change; the sections after it are fully written
  // before they are read in a launch.
  size_t off = 0;
  pl.ws_sync = off;  off += up256((size_t)units * DEC_SYNC_WORDS * 4);   // epoch, hint / appended-row slots (any M)
  pl.ws_hist = off;  off += M > 1 ? up256((size_t)units * M * hs * 8) : 0;          // tagged words
  pl.ws_part = off;  off += M > 1 ? up256((size_t)units * M * dec_part_stride(GT, d) * 8) : 0;
  pl.ws_D = off;     off += !pl.d_smem ? up256((size_t)units * M * dec_dchunk(pl.chunk) * 2) : 0;
  pl.ws_rows = off;  off += pl.rows_global ? up256((size_t)units * M * pl.R_cap * 4) : 0;
  pl.ws_total = off;
  return pl;
}

cudaError_t launch_decode(DecodeParams& p, const DecodePlan& pl, void* ws, int is_bf16, cudaStream_t s) {
  DecodeKernel kern = get_kernel(is_bf16, p.rbits / 32, pl.GT);
  if (!kern) return cudaErrorNotSupported;
  uint8_t* w = reinterpret_cast<uint8_t*>(ws);
  p.trace = decode_trace_buf();
#if HATA_DIAG
  { const char* e = std::getenv("HATA_DEBUG"); p.dbg = e ? std::atoi(e) : 0; }   // diagnostics build only
#else
  p.dbg = 0;
#endif
  p.use_hint = option_value(OPT_SELECTION_HINT);
  p.M = pl.M; p.stages = pl.stages; p.chunk = pl.chunk; p.nbins = pl.nbins; p.rows_cap = pl.rows_cap; p.R_cap = pl.R_cap;
  p.d_smem = pl.d_smem;
  p.ws_sync = reinterpret_cast<unsigned*>(w + pl.ws_sync);
  p.ws_hist = pl.M > 1 ? reinterpret_cast<uint64_t*>(w + pl.ws_hist) : nullptr;
  p.ws_part = pl.M > 1 ? reinterpret_cast<uint64_t*>(w + pl.ws_part) : nullptr;
  p.ws_D = !pl.d_smem ? reinterpret_cast<uint16_t*>(w + pl.ws_D) : nullptr;
  p.ws_rows = pl.rows_global ? reinterpret_cast<int32_t*>(w + pl.ws_rows) : nullptr;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[2];
  cfg.gridDim = dim3(pl.M, p.B * p.Hkv);
  cfg.blockDim = dim3(DEC_THREADS);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = s;
  // ranks of a unit meet at a spin barrier: they must be co-resident.  The
  // plan keeps the grid within one CTA per SM, so a plain launch is
  // co-resident as soon as the SMs are free; a cooperative launch guarantees
  // it, but then cannot start any CTA before every SM is free -- which rules
  // out overlapping the prologue (W_g, the code stream) with the preceding
  // kernel's tail under programmatic dependent launch (HATA_OPT_COOPERATIVE)
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = (pl.M > 1 && option_value(OPT_COOPERATIVE)) ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  // programmatic dependent launch: the prologue (barrier init, W_g loads)
  // overlaps the tail of the preceding kernel in the stream; the kernel waits
  // (griddepcontrol.wait) before touching anything that kernel may produce
  if (option_value(OPT_PDL)) {
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs = 2;
  }
  return cudaLaunchKernelEx(&cfg, kern, (const DecodeParams)p);
}

// ---------------------------------------------------------------- shard phase 3
typedef void (*PartialKernel)(const PartialParams);
template <typename T>
static PartialKernel pick_partial(int GT) {
  switch (GT) {
    case 1: return hata_partial_attn_kernel<T, 1, 128>;
    case 2: return hata_partial_attn_kernel<T, 2, 128>;
    case 4: return hata_partial_attn_kernel<T, 4, 128>;
    case 5: return hata_partial_attn_kernel<T, 5, 128>;
    case 8: return hata_partial_attn_kernel<T, 8, 128>;
  }
  return nullptr;
}

cudaError_t launch_partial_attn(PartialParams& p, int GT, int is_bf16, cudaStream_t s) {
  PartialKernel kern = is_bf16 ? pick_partial<__nv_bfloat16>(GT) : pick_partial<float>(GT);
  if (!kern) return cudaErrorNotSupported;
  if (p.splits < 1) return cudaErrorInvalidValue;
  const int eb = is_bf16 ? 2 : 4;
  const int rowb = p.d * eb + DEC_ROW_PAD;
  const int QS = dec_qstride(p.d);
  int rc = 192;
  if (rc > p.k) rc = p.k;
  p.rows_cap = rc;
  const size_t smem = ((2 * (size_t)rc * rowb + 127) & ~(size_t)127) + (size_t)GT * rc * 4 + (size_t)GT * QS * 4 +
                      32 * 4 + 16 + (size_t)GT * p.d * eb + (size_t)p.k * 4;
  if (smem > (size_t)SMEM_LIMIT) return cudaErrorNotSupported;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<dim3(p.splits, p.B * p.Hkv), DEC_THREADS, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace hata

namespace hata {
// process-wide options (hata_set_option); defaults on
static std::atomic<int> g_opts[OPT_COUNT] = {{1}, {1}, {0}};   // hint on, PDL on, cooperative off
int option_value(int opt) { return (opt >= 0 && opt < OPT_COUNT) ? g_opts[opt].load(std::memory_order_relaxed) : 0; }
void set_option_value(int opt, int v) { if (opt >= 0 && opt < OPT_COUNT) g_opts[opt].store(v, std::memory_order_relaxed); }

static unsigned long long* g_trace_buf = nullptr;   // host-side: copied into DecodeParams::trace
cudaError_t set_decode_trace(void* buf) {
  g_trace_buf = reinterpret_cast<unsigned long long*>(buf);
  return cudaSuccess;
}
unsigned long long* decode_trace_buf() { return g_trace_buf; }

static __global__ void timestamp_kernel(unsigned long long* dst) { *dst = globaltimer_ns(); }
cudaError_t launch_timestamp(void* dst, cudaStream_t s) {
  timestamp_kernel<<<1, 1, 0, s>>>(reinterpret_cast<unsigned long long*>(dst));
  return cudaGetLastError();
}
}  // namespace hata
