// Probe: how fast can 144 SMs pull a ~16.8 MB burst (one CFG-4 decode step of
// codes) from HBM?  Each CTA reads a contiguous slice; timestamps (globaltimer)
// at issue / first / last arrival are recorded per CTA.  Buffers rotate over a
// 1 GB region so no step hits in L2.  Not product code.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint64_t gtime() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(b))); }
__device__ __forceinline__ void expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(b)), "r"(n) : "memory"); }
__device__ __forceinline__ bool tryw(uint64_t* b, uint32_t ph) {
  uint32_t ok; asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(sa(b)), "r"(ph) : "memory"); return ok;
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(sa(d)), "l"(s), "r"(n), "r"(sa(b)) : "memory");
}

// mode 0: bulk copies of `stage` bytes, all issued at t0 by thread 0
// mode 1: every thread LDG.128 (ld.global.nc) its share, all loads in flight
__global__ void burst(const uint8_t* base, size_t per_cta, int stage, int mode, uint64_t* ts, uint32_t* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bars[64];
  const uint8_t* src = base + (size_t)blockIdx.x * per_cta;
  const int nst = (int)((per_cta + stage - 1) / stage);
  uint64_t t0 = gtime();
  if (mode == 0) {
    if (threadIdx.x == 0) { for (int s = 0; s < nst; ++s) mbar_init(&bars[s]); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    if (threadIdx.x == 0) {
      t0 = gtime();
      for (int s = 0; s < nst; ++s) { uint32_t n = (uint32_t)min((size_t)stage, per_cta - (size_t)s * stage); expect(&bars[s], n); bulk(sm + (size_t)s * stage, src + (size_t)s * stage, n, &bars[s]); }
      uint64_t tf = 0;
      for (int s = 0; s < nst; ++s) { while (!tryw(&bars[s], 0)) {} if (s == 0) tf = gtime(); }
      uint64_t tl = gtime();
      ts[blockIdx.x * 3 + 0] = t0; ts[blockIdx.x * 3 + 1] = tf; ts[blockIdx.x * 3 + 2] = tl;
    }
  } else {
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    const int n16 = (int)(per_cta / 16);
    uint32_t acc = 0;
    __syncthreads();
    t0 = gtime();
    constexpr int U = 16;
    for (int i = threadIdx.x; i < n16; i += blockDim.x * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) { int j = i + u * blockDim.x; if (j < n16) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(s4 + j)); else v[u] = make_uint4(0,0,0,0); }
#pragma unroll
      for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].w;
    }
    __syncthreads();
    if (threadIdx.x == 0) { uint64_t tl = gtime(); ts[blockIdx.x * 3 + 0] = t0; ts[blockIdx.x * 3 + 1] = tl; ts[blockIdx.x * 3 + 2] = tl; }
    if (acc == 0x1234567) sink[0] = acc;
  }
}

int main() {
  const size_t total = (size_t)1 << 30;
  uint8_t* buf; CK(cudaMalloc(&buf, total)); CK(cudaMemset(buf, 3, total));
  uint64_t* ts; CK(cudaMalloc(&ts, 4096 * 8 * 3)); uint32_t* sink; CK(cudaMalloc(&sink, 64));
  cudaFuncSetAttribute(burst, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  std::vector<uint64_t> h(4096 * 3);
  struct Cfg { int grid; size_t per; int stage; int mode; int threads; };
  std::vector<Cfg> cfgs = {
    {144, 117 * 1024, 16384, 0, 512}, {144, 117 * 1024, 8192, 0, 512}, {144, 117 * 1024, 32768, 0, 512},
    {144, 117 * 1024, 4096, 0, 512}, {144, 117 * 1024, 0, 1, 512}, {144, 117 * 1024, 0, 1, 1024},
    {148, 114 * 1024, 16384, 0, 512}, {144, 58 * 1024, 16384, 0, 512}, {144, 29 * 1024, 8192, 0, 512},
    {144, 190 * 1024, 16384, 0, 512}, {72, 117 * 1024, 16384, 0, 512}, {288, 58 * 1024, 16384, 1, 512},
  };
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (auto c : cfgs) {
    size_t step = (size_t)c.grid * c.per;
    int nrot = (int)(total / step);
    std::vector<double> first, last, wall;
    for (int it = 0; it < 24; ++it) {
      const uint8_t* b = buf + (size_t)(it % nrot) * step;
      cudaEventRecord(e0);
      burst<<<c.grid, c.threads, c.mode == 0 ? 200 * 1024 : 0>>>(b, c.per, c.stage > 0 ? c.stage : 16384, c.mode, ts, sink);
      cudaEventRecord(e1);
      CK(cudaDeviceSynchronize());
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      CK(cudaMemcpy(h.data(), ts, c.grid * 24, cudaMemcpyDeviceToHost));
      uint64_t tmin = ~0ull, fmax = 0, lmax = 0; std::vector<double> f;
      for (int i = 0; i < c.grid; ++i) { tmin = std::min(tmin, h[i * 3]); }
      for (int i = 0; i < c.grid; ++i) { fmax = std::max(fmax, h[i * 3 + 1]); lmax = std::max(lmax, h[i * 3 + 2]); f.push_back((double)(h[i * 3 + 1] - tmin)); }
      std::sort(f.begin(), f.end());
      if (it >= 4) { first.push_back(f[f.size() / 2] / 1e3); last.push_back((lmax - tmin) / 1e3); wall.push_back(ms * 1e3); }
    }
    std::sort(first.begin(), first.end()); std::sort(last.begin(), last.end()); std::sort(wall.begin(), wall.end());
    double l = last[last.size() / 2];
    printf("{\"grid\":%d,\"per_cta_KB\":%zu,\"stage\":%d,\"mode\":\"%s\",\"threads\":%d,\"MB\":%.1f,\"first_med_us\":%.2f,\"last_us\":%.2f,\"GBps_inkernel\":%.0f,\"event_us\":%.2f}\n",
           c.grid, c.per / 1024, c.stage, c.mode == 0 ? "bulk" : "ldg", c.threads, step / 1e6, first[first.size() / 2], l, step / (l * 1e-6) / 1e9, wall[wall.size() / 2]);
  }
  return 0;
}
