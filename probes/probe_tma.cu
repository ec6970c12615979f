// Probe: cost of ISSUING cp.async.bulk (TMA) requests, per request size, on
// a busy chip (all 144 CTAs issuing at once), and completion times.  Also the
// LDG.128 alternative for a 32 KB block.  Not product code.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// mode 0: thread 0 issues all N copies of S bytes; mode 1: lanes of warp 0 share the issuing;
// mode 2: 16 warps' lane 0 share; mode 3: LDG.128 by all threads (no TMA)
__global__ void k_issue(const uint8_t* src, size_t per_cta, int S, int mode, uint64_t* ts, uint32_t* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar;
  const uint8_t* s = src + (size_t)blockIdx.x * per_cta;
  const int N = (int)(per_cta / S);
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  uint64_t t0 = gt(), t1 = 0;
  if (mode < 3) {
    if (threadIdx.x == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&bar)), "r"((uint32_t)(N * S)) : "memory");
    __syncthreads();
    int nissuers = mode == 0 ? 1 : (mode == 1 ? 32 : 16);
    int me = mode == 0 ? (threadIdx.x == 0 ? 0 : -1) : (mode == 1 ? (threadIdx.x < 32 ? threadIdx.x : -1) : ((threadIdx.x & 31) == 0 ? threadIdx.x / 32 : -1));
    if (me >= 0)
      for (int i = me; i < N; i += nissuers)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(sa(sm + (size_t)i * S)), "l"(s + (size_t)i * S), "r"(S), "r"(sa(&bar)) : "memory");
    if (threadIdx.x == 0) t1 = gt();
    uint32_t ok = 0;
    while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(sa(&bar)) : "memory");
  } else {
    const uint4* s4 = reinterpret_cast<const uint4*>(s);
    const int n16 = (int)(per_cta / 16);
    for (int i = threadIdx.x; i < n16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = __ldg(s4 + i);
    if (threadIdx.x == 0) t1 = gt();
  }
  __syncthreads();
  if (threadIdx.x == 0) { ts[blockIdx.x * 3] = t0; ts[blockIdx.x * 3 + 1] = t1; ts[blockIdx.x * 3 + 2] = gt(); }
  if (sm[threadIdx.x * 7] == 0xEE) sink[0] = 1;
}

int main() {
  const size_t total = (size_t)1 << 30;
  uint8_t* buf; CK(cudaMalloc(&buf, total)); CK(cudaMemset(buf, 5, total));
  uint64_t* ts; CK(cudaMalloc(&ts, 4096 * 24)); uint32_t* sink; CK(cudaMalloc(&sink, 64));
  cudaFuncSetAttribute(k_issue, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct C { size_t per; int S; int mode; };
  std::vector<C> cs = {{131072, 16384, 0}, {131072, 65536, 0}, {131072, 4096, 0}, {131072, 4096, 1}, {131072, 1024, 1},
                       {32768, 256, 0}, {32768, 256, 1}, {32768, 256, 2}, {32768, 32768, 0}, {32768, 0, 3}, {58368, 256, 1}, {58368, 256, 2}};
  const int grid = 144;
  for (auto c : cs) {
    std::vector<double> iss, done;
    for (int rep = 0; rep < 14; ++rep) {
      const uint8_t* b = buf + (size_t)(rep % 40) * grid * c.per;
      k_issue<<<grid, 512, 200 * 1024>>>(b, c.per, c.S > 0 ? c.S : 16, c.mode, ts, sink); CK(cudaDeviceSynchronize());
      std::vector<uint64_t> h(grid * 3); CK(cudaMemcpy(h.data(), ts, grid * 24, cudaMemcpyDeviceToHost));
      uint64_t tmin = ~0ull; for (int i = 0; i < grid; ++i) tmin = std::min(tmin, h[3 * i]);
      std::vector<double> a, d; for (int i = 0; i < grid; ++i) { a.push_back((h[3 * i + 1] - h[3 * i]) / 1e3); d.push_back((h[3 * i + 2] - tmin) / 1e3); }
      std::sort(a.begin(), a.end()); std::sort(d.begin(), d.end());
      if (rep >= 4) { iss.push_back(a[a.size() / 2]); done.push_back(d.back()); }
    }
    std::sort(iss.begin(), iss.end()); std::sort(done.begin(), done.end());
    const char* mn[] = {"thread0", "warp0_lanes", "16warps_lane0", "ldg128_all"};
    printf("{\"per_cta\":%zu,\"req_bytes\":%d,\"issuer\":\"%s\",\"issue_us\":%.2f,\"all_done_us\":%.2f}\n", c.per, c.S, mn[c.mode], iss[iss.size() / 2], done[done.size() / 2]);
  }
  return 0;
}
