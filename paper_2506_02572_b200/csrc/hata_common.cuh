// Shared device helpers for the HATA sm_100a kernels (product path only; the
// CPU oracle in oracle/ shares nothing with this file).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cooperative_groups.h>
#include <stdint.h>

namespace hata {

namespace cg = cooperative_groups;

// ---------------------------------------------------------------- elements
template <typename T> struct Elem;
template <> struct Elem<float> {
  static constexpr int bytes = 4;
  __device__ static __forceinline__ float to_f(float x) { return x; }
  __device__ static __forceinline__ float from_f(float x) { return x; }
};
template <> struct Elem<__nv_bfloat16> {
  static constexpr int bytes = 2;
  __device__ static __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
  __device__ static __forceinline__ __nv_bfloat16 from_f(float x) { return __float2bfloat16_rn(x); }
};

// Load EPL consecutive elements (EPL*sizeof(T) bytes, naturally aligned) as floats.
template <typename T, int EPL>
__device__ __forceinline__ void load_row_slice(const T* __restrict__ p, float (&v)[EPL]) {
  if constexpr (sizeof(T) == 2) {
    static_assert(EPL % 2 == 0, "bf16 slice must be even");
    if constexpr (EPL == 8) {
      uint4 r = __ldg(reinterpret_cast<const uint4*>(p));
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
      for (int i = 0; i < 4; ++i) { float2 f = __bfloat1622float2(h[i]); v[2 * i] = f.x; v[2 * i + 1] = f.y; }
    } else if constexpr (EPL == 4) {
      uint2 r = __ldg(reinterpret_cast<const uint2*>(p));
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
      for (int i = 0; i < 2; ++i) { float2 f = __bfloat1622float2(h[i]); v[2 * i] = f.x; v[2 * i + 1] = f.y; }
    } else {
      uint32_t r = __ldg(reinterpret_cast<const uint32_t*>(p));
      float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r));
      v[0] = f.x; v[1] = f.y;
    }
  } else {
    if constexpr (EPL % 4 == 0) {
#pragma unroll
      for (int i = 0; i < EPL / 4; ++i) {
        float4 r = __ldg(reinterpret_cast<const float4*>(p) + i);
        v[4 * i] = r.x; v[4 * i + 1] = r.y; v[4 * i + 2] = r.z; v[4 * i + 3] = r.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < EPL; ++i) v[i] = __ldg(p + i);
    }
  }
}

// ---------------------------------------------------------------- mbarrier / bulk copy (TMA engine)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// 16-byte cp.async global -> shared (L2-only caching)
__device__ __forceinline__ void cp_async16_g(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  while (!mbar_try_wait(b, parity)) {
  }
}
// cp.async.bulk global -> shared (this CTA), completion signalled on mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Programmatic dependent launch (griddepcontrol): wait for the preceding
// grid's completion + memory flush; allow the dependent grid to launch.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Bitwise select: k ? b : a  (one LOP3).
__device__ __forceinline__ uint32_t lop_mux(uint32_t k, uint32_t b, uint32_t a) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xCA;" : "=r"(r) : "r"(k), "r"(b), "r"(a));
  return r;
}
// Full adder on 32 bit lanes: s = a^b^c, cy = maj(a,b,c).
__device__ __forceinline__ void full_add(uint32_t a, uint32_t b, uint32_t c, uint32_t& s, uint32_t& cy) {
  asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(s) : "r"(a), "r"(b), "r"(c));
  asm("lop3.b32 %0, %1, %2, %3, 0xE8;" : "=r"(cy) : "r"(a), "r"(b), "r"(c));
}

// ---------------------------------------------------------------- warp-level tensor core (HMMA)
// D += A(16x16, row) * B(16x8, col), bf16 inputs, fp32 accumulate.
// Fragment ownership (gid = lane / 4, tig = lane % 4):
//   a0: A[gid][2tig..2tig+1]   a1: A[gid+8][2tig..]   a2: A[gid][8+2tig..]   a3: A[gid+8][8+2tig..]
//   b0: B[2tig..2tig+1][gid]   b1: B[8+2tig..][gid]
//   d0,d1: D[gid][2tig, 2tig+1]   d2,d3: D[gid+8][2tig, 2tig+1]
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// Two 8x8 b16 tiles, transposed: lanes 0-7 give the row addresses of tile 0,
// lanes 8-15 those of tile 1 (16-byte rows).  Yields a B fragment (b0, b1)
// from a row-major [k][n] smem matrix.
__device__ __forceinline__ void ldsm_x2_trans(uint32_t& r0, uint32_t& r1, const void* row) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];"
               : "=r"(r0), "=r"(r1)
               : "r"(smem_u32(row)));
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace hata
