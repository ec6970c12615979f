// Probe: cost of a "phase" of cold code (first execution in a launch) vs the
// same phase warm (second pass in the same launch), on a full chip (144 CTAs
// x 256 threads, 1 CTA/SM), for phase-structured code like the decode
// kernel's: NPH distinct phases, each = 8 independent ALU chains (ILP), a
// barrier, a lane-dependent branch and a short runtime loop.  Thread 0 stamps
// %globaltimer at every phase boundary.  Not product code.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <int K, int NOPS>
__device__ __forceinline__ void phase(uint32_t (&v)[8], int n, uint32_t* sm) {
#pragma unroll
  for (int i = 0; i < NOPS; ++i)
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = (v[c] ^ (0x9e3779b9u * (K + 1) + c)) + (v[(c + 1) & 7] >> ((K + i) & 15));
  __syncthreads();
  if (threadIdx.x < 32 * (K % 8 + 1)) {
#pragma unroll
    for (int c = 0; c < 2; ++c) v[c] = __funnelshift_l(v[c], v[(c + 3) & 7], K + c);
  }
#pragma unroll 1
  for (int i = 0; i < n; ++i) v[i & 7] += sm[(threadIdx.x + i * (K + 1)) & 255];
  sm[threadIdx.x] = v[K & 7];
  __syncthreads();
}

template <int K, int NOPS>
__device__ __forceinline__ void phases(uint32_t (&v)[8], int n, uint32_t* sm, unsigned long long* st) {
  if constexpr (K > 0) {
    phases<K - 1, NOPS>(v, n, sm, st);
    phase<K, NOPS>(v, n, sm);
    if (threadIdx.x == 0) st[K] = gtime();
  }
}

template <int NPH, int NOPS>
__global__ void __launch_bounds__(256, 1) k_phase(unsigned long long* out, uint32_t* sink, int n) {
  __shared__ uint32_t sm[256];
  __shared__ unsigned long long st[2][NPH + 1];
  uint32_t v[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) v[c] = threadIdx.x * (c + 1) + blockIdx.x;
  sm[threadIdx.x] = v[0];
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    if (threadIdx.x == 0) st[pass][0] = gtime();
    phases<NPH, NOPS>(v, n, sm, st[pass]);
  }
  if (threadIdx.x == 0) {
    out[blockIdx.x * 2] = st[0][NPH] - st[0][0];
    out[blockIdx.x * 2 + 1] = st[1][NPH] - st[1][0];
  }
  uint32_t x = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) x ^= v[c];
  if (x == 0x12345u) sink[0] = x;
}

template <int NPH, int NOPS>
static void run(const char* name) {
  const int G = 144;
  unsigned long long* d;
  uint32_t* s;
  cudaMalloc(&d, G * 2 * 8);
  cudaMalloc(&s, 4);
  std::vector<unsigned long long> h(G * 2);
  for (int rep = 0; rep < 3; ++rep) {
    k_phase<NPH, NOPS><<<G, 256>>>(d, s, 6);
    cudaDeviceSynchronize();
    cudaMemcpy(h.data(), d, G * 2 * 8, cudaMemcpyDeviceToHost);
    std::vector<double> a, b;
    for (int i = 0; i < G; ++i) { a.push_back(h[2 * i] / 1e3); b.push_back(h[2 * i + 1] / 1e3); }
    std::sort(a.begin(), a.end());
    std::sort(b.begin(), b.end());
    printf("{\"probe\":\"phase\",\"variant\":\"%s\",\"phases\":%d,\"ops\":%d,\"rep\":%d,\"cold_us_med\":%.3f,\"warm_us_med\":%.3f,"
           "\"cold_per_phase_us\":%.3f,\"warm_per_phase_us\":%.3f}\n",
           name, NPH, NOPS, rep, a[G / 2], b[G / 2], a[G / 2] / NPH, b[G / 2] / NPH);
  }
  cudaFree(d);
  cudaFree(s);
}

int main() {
  run<16, 2>("fits_l15");     // code < 32 KB: the second pass runs from the L1.5 I-cache
  run<64, 2>("exceeds_l15");  // same phases, 4x the code: the second pass refetches from L2
  run<16, 16>("fits_big");
  run<64, 16>("exceeds_big");
  return 0;
}
