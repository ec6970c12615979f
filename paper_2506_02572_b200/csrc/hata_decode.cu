// Host-side planning + dispatch of the fused decode kernel (hata_decode.cuh).
#include <cstdlib>
#include <mutex>
#include "hata_internal.h"
#include "hata_decode.cuh"

namespace hata {

int device_sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

static int group_template(int G) {
  if (G <= 1) return 1;
  if (G <= 2) return 2;
  if (G <= 4) return 4;
  if (G <= 5) return 5;
  if (G <= 8) return 8;
  return -1;
}

typedef void (*DecodeKernel)(const DecodeParams);

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
static DecodeKernel get_kernel(int is_bf16, int W, int GT) {
  return is_bf16 ? pick_w<__nv_bfloat16>(W, GT) : pick_w<float>(W, GT);
}

static DecodeParams shape_params(int B, int Hq, int Hkv, int d, int rbits, int C, int chunk, int rows_cap, bool gD,
                                 bool gsel) {
  DecodeParams p = {};
  p.B = B; p.Hq = Hq; p.Hkv = Hkv; p.G = Hq / Hkv; p.d = d; p.rbits = rbits;
  p.C = C; p.chunk = chunk; p.rows_cap = rows_cap; p.nbins = p.G * rbits + 1;
  p.gD = gD ? reinterpret_cast<uint16_t*>(16) : nullptr;     // non-null marker for layout only
  p.gsel = gsel ? reinterpret_cast<int32_t*>(16) : nullptr;
  return p;
}

DecodePlan plan_decode(int B, int Hq, int Hkv, int d, int rbits, int64_t n_max, int k, int elem_bytes) {
  DecodePlan pl = {};
  const int G = Hq / Hkv;
  pl.GT = group_template(G);
  pl.nbins = G * rbits + 1;
  const int units = B * Hkv;
  int C = device_sm_count() / (units > 0 ? units : 1);
  if (C > 16) C = 16;
  if (C < 1) C = 1;
  const int64_t by_len = (n_max + 1023) / 1024;
  if (by_len < C) C = (int)(by_len < 1 ? 1 : by_len);
  if (const char* e = std::getenv("HATA_CLUSTER")) {
    int v = std::atoi(e);
    if (v >= 1 && v <= 16) C = v;
  }
  const int W = rbits / 32;
  DecodeKernel kern = get_kernel(elem_bytes == 2, W, pl.GT);
  for (;;) {
    int64_t per = (n_max + C - 1) / C;
    pl.C = C;
    pl.chunk = (int)((per + DEC_CHUNK_ALIGN - 1) / DEC_CHUNK_ALIGN * DEC_CHUNK_ALIGN);
    if (pl.chunk < DEC_CHUNK_ALIGN) pl.chunk = DEC_CHUNK_ALIGN;
    const int64_t kmax = k < n_max ? k : n_max;
    pl.rows_cap = (int)((kmax + C - 1) / C);
    if (pl.rows_cap < 1) pl.rows_cap = 1;
    pl.gD = pl.chunk > DEC_D_SMEM_MAX;
    pl.gsel = pl.rows_cap > DEC_SEL_SMEM_MAX;
    DecodeParams sp = shape_params(B, Hq, Hkv, d, rbits, C, pl.chunk, pl.rows_cap, pl.gD, pl.gsel);
    pl.smem = decode_smem_layout(sp, pl.GT > 0 ? pl.GT : 1, elem_bytes).total;
    bool ok = true;
    if (kern && C > 1) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem);
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      cfg.gridDim = dim3(C, units);
      cfg.blockDim = dim3(DEC_THREADS);
      cfg.dynamicSmemBytes = pl.smem;
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      int ncl = 0;
      // an error here means "no device to ask" (CPU-only build host): keep C
      if (cudaOccupancyMaxActiveClusters(&ncl, (void*)kern, &cfg) == cudaSuccess && ncl < 1) ok = false;
      cudaGetLastError();
    }
    if (ok || C == 1) break;
    C = C > 8 ? 8 : C / 2;
  }
  pl.ws_D = pl.gD ? ((size_t)units * pl.C * pl.chunk * 2 + 255) / 256 * 256 : 0;
  pl.ws_sel = pl.gsel ? ((size_t)units * pl.C * pl.rows_cap * 4 + 255) / 256 * 256 : 0;
  pl.ws_total = pl.ws_D + pl.ws_sel;
  return pl;
}

cudaError_t launch_decode(DecodeParams& p, const DecodePlan& pl, int is_bf16, cudaStream_t s) {
  DecodeKernel kern = get_kernel(is_bf16, p.rbits / 32, pl.GT);
  if (!kern) return cudaErrorNotSupported;
  p.C = pl.C; p.chunk = pl.chunk; p.rows_cap = pl.rows_cap; p.nbins = pl.nbins;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem);
  if (e != cudaSuccess) return e;
  if (pl.C > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[2];
  cfg.gridDim = dim3(pl.C, p.B * p.Hkv);
  cfg.blockDim = dim3(DEC_THREADS);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = s;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = pl.C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, (const DecodeParams)p);
}

}  // namespace hata
