// HashEncode kernels: decode-time append (Alg. 3 lines 2-9) and the CUDA-core
// prefill key hash (Alg. 1 lines 2-5) used for fp32 caches and as the
// fallback shape path.  The bf16 prefill path runs on tcgen05 (hata_hash_tc.cu).
//
// PAPER: Alg. 2 HashEncode: Sign(MatMul(V, W_H)) -> BitPack.
//        Alg. 3 lines 3-9; §4 "Kernel fusion for hash encoding".
#include "hata_internal.h"
#include "hata_common.cuh"

namespace hata {

// One CTA per (b, g): write K/V rows at pos[b] and the packed code of k_new.
template <typename T>
__global__ void __launch_bounds__(256) append_kernel(AppendParams p) {
  __shared__ float x[1024];
  const int bg = blockIdx.x, b = bg / p.Hkv, g = bg % p.Hkv;
  const int64_t pos = p.pos[b];
  if (pos < 0 || pos >= p.cap) return;  // device-side capacity guard (ABI: caller error)
  const T* kn = reinterpret_cast<const T*>(p.k_new) + (int64_t)bg * p.d;
  const T* vn = reinterpret_cast<const T*>(p.v_new) + (int64_t)bg * p.d;
  T* Kd = reinterpret_cast<T*>(p.K) + (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh + pos * p.kv_st;
  T* Vd = reinterpret_cast<T*>(p.V) + (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh + pos * p.kv_st;
  for (int i = threadIdx.x; i < p.d; i += blockDim.x) {
    T kv = kn[i];
    Kd[i] = kv;
    Vd[i] = vn[i];
    x[i] = Elem<T>::to_f(kv);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int W = p.rbits / 32;
  const T* Wg = reinterpret_cast<const T*>(p.Wh) + (int64_t)g * p.d * p.rbits;
  uint32_t* cd = p.codes + (int64_t)b * p.c_sb + (int64_t)g * p.c_sh + pos * W;
  for (int w = warp; w < W; w += blockDim.x / 32) {
    float acc = 0.f;
    const T* col = Wg + w * 32 + lane;
#pragma unroll 8
    for (int j = 0; j < p.d; ++j) acc = fmaf(x[j], Elem<T>::to_f(col[(int64_t)j * p.rbits]), acc);
    const uint32_t word = __ballot_sync(0xffffffffu, acc >= 0.f);
    if (lane == 0) cd[w] = word;
  }
  // the appended rows are visible GPU-wide before a dependent decode launch
  // (which streams code rows before its griddepcontrol.wait) may start: every
  // writer fences, then the CTA syncs, then triggers (a CTA counts as
  // triggered as soon as any of its threads executes the trigger)
  __threadfence();
  __syncthreads();
  griddep_launch_dependents();
}

// CUDA-core key hashing: CTA = 64 tokens x all words of one (b, g).
// Thread (token, word) accumulates 32 projections in fp32 (j ascending).
template <typename T>
__global__ void __launch_bounds__(256) hash_keys_simt_kernel(HashKeysParams p) {
  extern __shared__ __align__(16) float sm[];
  const int W = p.rbits / 32;
  const int TOK = 256 / W;                    // tokens per CTA
  float* xs = sm;                             // [TOK][d+1]
  float* ws = sm + TOK * (p.d + 1);           // [d][rbits]
  const int bg = blockIdx.y, b = bg / p.Hkv, g = bg % p.Hkv;
  const int64_t tbase = p.t0 + (int64_t)blockIdx.x * TOK;
  const T* Kb = reinterpret_cast<const T*>(p.K) + (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh;
  const T* Wg = reinterpret_cast<const T*>(p.Wh) + (int64_t)g * p.d * p.rbits;
  for (int i = threadIdx.x; i < p.d * p.rbits; i += blockDim.x) ws[i] = Elem<T>::to_f(Wg[i]);
  for (int i = threadIdx.x; i < TOK * p.d; i += blockDim.x) {
    const int tk = i / p.d, j = i % p.d;
    const int64_t t = tbase + tk;
    xs[tk * (p.d + 1) + j] = (t < p.t0 + p.n) ? Elem<T>::to_f(Kb[t * p.kv_st + j]) : 0.f;
  }
  __syncthreads();
  const int tk = threadIdx.x / W, w = threadIdx.x % W;
  const int64_t t = tbase + tk;
  if (tk < TOK && t < p.t0 + p.n) {
  float acc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = 0.f;
  const float* xr = xs + tk * (p.d + 1);
  for (int j = 0; j < p.d; ++j) {
    const float xv = xr[j];
    const float4* wr = reinterpret_cast<const float4*>(ws + j * p.rbits + w * 32);
#pragma unroll
    for (int q4 = 0; q4 < 8; ++q4) {
      const float4 wv = wr[q4];
      acc[4 * q4 + 0] = fmaf(xv, wv.x, acc[4 * q4 + 0]);
      acc[4 * q4 + 1] = fmaf(xv, wv.y, acc[4 * q4 + 1]);
      acc[4 * q4 + 2] = fmaf(xv, wv.z, acc[4 * q4 + 2]);
      acc[4 * q4 + 3] = fmaf(xv, wv.w, acc[4 * q4 + 3]);
    }
  }
  uint32_t word = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) word |= (acc[i] >= 0.f ? 1u : 0u) << i;
  p.codes[(int64_t)b * p.c_sb + (int64_t)g * p.c_sh + t * W + w] = word;
  }
  __threadfence();                          // codes visible before dependents start (see append_kernel)
  __syncthreads();
  griddep_launch_dependents();
}

cudaError_t launch_append(const AppendParams& p, int is_bf16, cudaStream_t s) {
  dim3 grid(p.B * p.Hkv);
  if (is_bf16) append_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(p);
  else append_kernel<float><<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_hash_keys_simt(const HashKeysParams& p, int is_bf16, cudaStream_t s) {
  const int W = p.rbits / 32;
  const int TOK = 256 / W;
  const size_t smem = ((size_t)TOK * (p.d + 1) + (size_t)p.d * p.rbits) * 4;
  dim3 grid((unsigned)((p.n + TOK - 1) / TOK), p.B * p.Hkv);
  if (p.n == 0) return cudaSuccess;
  if (is_bf16) {
    cudaFuncSetAttribute(hash_keys_simt_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    hash_keys_simt_kernel<__nv_bfloat16><<<grid, 256, smem, s>>>(p);
  } else {
    cudaFuncSetAttribute(hash_keys_simt_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    hash_keys_simt_kernel<float><<<grid, 256, smem, s>>>(p);
  }
  return cudaGetLastError();
}

}  // namespace hata
