// Probe: latencies / throughputs that shape the decode tail on sm_100a.
//  1. mma.sync m16n8k16 bf16 dependent-chain latency and per-SM throughput
//  2. shfl / smem load latency chains
//  3. gather of 114 random 256-byte rows (K and V) per SM from a 512 MB cache:
//     16-byte cp.async vs one cp.async.bulk per row vs LDG.128 into registers
// Not product code.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_mma_chain(int iters, float* out, long long* cyc) {
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3, 7u, 9u}, b0 = threadIdx.x ^ 5, b1 = 11;
  float c[4] = {0, 0, 0, 0};
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = c[0] + c[1] + c[2] + c[3];
}
__global__ void k_mma_tput(int iters, float* out, long long* cyc) {
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3, 7u, 9u}, b0 = threadIdx.x ^ 5, b1 = 11;
  float c[8][4] = {};
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  float s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_shfl_chain(int iters, int* out, long long* cyc) {
  int v = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1) + 1;
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = v;
}
__global__ void k_lds_chain(int iters, int* out, long long* cyc) {
  __shared__ int s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i * 7 + 1) & 1023;
  __syncthreads();
  int v = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = s[v];
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = v;
}
__global__ void k_sync_chain(int iters, int* out, long long* cyc) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// gather: each CTA fetches R random rows (256 B) from K and from V
__global__ void k_gather(const uint8_t* K, const uint8_t* V, const int* rows, int R, int mode, uint64_t* ts, uint32_t* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar;
  const int rowb = 272;
  const int* myrows = rows + blockIdx.x * R;
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  uint64_t t0 = gt();
  if (mode == 0) {          // 16-byte cp.async
    const int col = threadIdx.x % 32, which = col / 16, ch = col % 16;
    const uint8_t* base = (which ? V : K) + ch * 16;
    uint8_t* dst = sm + which * R * rowb + ch * 16;
    for (int i = threadIdx.x / 32; i < R; i += blockDim.x / 32)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(sa(dst + i * rowb)), "l"(base + (size_t)myrows[i] * 256) : "memory");
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (mode == 1) {   // one bulk copy per row
    if (threadIdx.x == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&bar)), "r"(R * 512) : "memory");
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * R; i += blockDim.x) {
      const int which = i / R, rr = i % R;
      const uint8_t* src = (which ? V : K) + (size_t)myrows[rr] * 256;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];" :: "r"(sa(sm + which * R * rowb + rr * rowb)), "l"(src), "r"(sa(&bar)) : "memory");
    }
    uint32_t ok = 0;
    while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(sa(&bar)) : "memory");
  } else {                  // LDG.128 into registers then STS
    const int col = threadIdx.x % 32, which = col / 16, ch = col % 16;
    const uint8_t* base = (which ? V : K) + ch * 16;
    uint4 v[8];
    int n = 0;
    for (int i = threadIdx.x / 32; i < R && n < 8; i += blockDim.x / 32, ++n) v[n] = __ldg(reinterpret_cast<const uint4*>(base + (size_t)myrows[i] * 256));
    n = 0;
    for (int i = threadIdx.x / 32; i < R && n < 8; i += blockDim.x / 32, ++n) *reinterpret_cast<uint4*>(sm + which * R * rowb + i * rowb + ch * 16) = v[n];
  }
  __syncthreads();
  if (threadIdx.x == 0) { ts[blockIdx.x * 2] = t0; ts[blockIdx.x * 2 + 1] = gt(); }
  if (sm[threadIdx.x] == 0xAB && sm[3000] == 0xCD) sink[0] = 1;
}

int main() {
  float* fo; int* io; long long* cyc; CK(cudaMalloc(&fo, 1 << 22)); CK(cudaMalloc(&io, 1 << 22)); CK(cudaMalloc(&cyc, 8 * 4096));
  std::vector<long long> h(4096);
  auto med = [&](int n) { std::vector<long long> v(h.begin(), h.begin() + n); std::sort(v.begin(), v.end()); return (double)v[n / 2]; };
  const int it = 4096;
  k_mma_chain<<<148, 32>>>(it, fo, cyc); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost));
  printf("{\"probe\":\"mma_chain\",\"cyc_per_mma\":%.1f}\n", med(148) / it);
  for (int w : {1, 4, 8, 16}) {
    k_mma_tput<<<148, 32 * w>>>(it / 8, fo, cyc); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost));
    printf("{\"probe\":\"mma_tput\",\"warps\":%d,\"cyc_per_mma_per_warp\":%.2f,\"sm_mma_per_cyc\":%.3f}\n", w, med(148) / it, w * it / med(148));
  }
  k_shfl_chain<<<148, 32>>>(it, io, cyc); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost));
  printf("{\"probe\":\"shfl_chain\",\"cyc\":%.1f}\n", med(148) / it);
  k_lds_chain<<<148, 32>>>(it, io, cyc); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost));
  printf("{\"probe\":\"lds_chain\",\"cyc\":%.1f}\n", med(148) / it);
  for (int nt : {256, 512}) {
    k_sync_chain<<<148, nt>>>(it, io, cyc); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost));
    printf("{\"probe\":\"syncthreads\",\"threads\":%d,\"cyc\":%.1f}\n", nt, med(148) / it);
  }
  // gather
  const size_t rows_total = (size_t)1 << 21;     // 2M rows x 256 B = 512 MB per tensor
  uint8_t *K, *V; CK(cudaMalloc(&K, rows_total * 256)); CK(cudaMalloc(&V, rows_total * 256));
  CK(cudaMemset(K, 1, rows_total * 256)); CK(cudaMemset(V, 2, rows_total * 256));
  const int grid = 144;
  uint64_t* ts; CK(cudaMalloc(&ts, 4096 * 16)); uint32_t* sink; CK(cudaMalloc(&sink, 64));
  cudaFuncSetAttribute(k_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int R : {57, 114, 228}) {
    std::vector<int> hr(grid * R);
    int* dr; CK(cudaMalloc(&dr, grid * R * 4 * 16));
    for (int mode = 0; mode < 3; ++mode) {
      std::vector<double> tt;
      for (int rep = 0; rep < 12; ++rep) {
        uint32_t s = 12345 + rep * 777 + mode;
        for (auto& x : hr) { s = s * 1664525u + 1013904223u; x = (int)((s >> 8) % rows_total); }
        std::sort(hr.begin(), hr.end());
        CK(cudaMemcpy(dr, hr.data(), hr.size() * 4, cudaMemcpyHostToDevice));
        k_gather<<<grid, 512, 2 * R * 272>>>(K, V, dr, R, mode, ts, sink); CK(cudaDeviceSynchronize());
        std::vector<uint64_t> ht(grid * 2); CK(cudaMemcpy(ht.data(), ts, grid * 16, cudaMemcpyDeviceToHost));
        uint64_t t0 = ~0ull, t1 = 0; for (int i = 0; i < grid; ++i) { t0 = std::min(t0, ht[2 * i]); t1 = std::max(t1, ht[2 * i + 1]); }
        if (rep >= 2) tt.push_back((t1 - t0) / 1e3);
      }
      std::sort(tt.begin(), tt.end());
      const char* nm[] = {"cp.async16", "bulk_per_row", "ldg128"};
      printf("{\"probe\":\"gather\",\"rows_per_cta\":%d,\"mode\":\"%s\",\"us\":%.2f,\"GBps\":%.0f}\n", R, nm[mode], tt[tt.size() / 2],
             grid * R * 512.0 / (tt[tt.size() / 2] * 1e-6) / 1e9);
    }
  }
  return 0;
}
