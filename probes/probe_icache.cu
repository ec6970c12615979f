// Probe: cost of executing COLD straight-line code (instruction-cache misses)
// vs the same code warm, on a full chip (144 CTAs x 512 threads, 1 CTA/SM).
// The body is NI independent-ish ALU instructions emitted by the preprocessor;
// it is executed twice per launch and each pass is timed with clock64 by
// thread 0.  Also: the same with a __syncthreads every 64 instructions
// (phase-structured code).  Not product code.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define R4(x) x x x x
#define R16(x) R4(R4(x))
#define R64(x) R16(R4(x))
#define R256(x) R64(R4(x))
#define R1024(x) R256(R4(x))

#define OPS asm volatile("add.u32 %0, %0, %1;\n\txor.b32 %1, %1, %0;" : "+r"(a), "+r"(b));
#define OPS_SYNC R16(OPS) __syncthreads();

template <int MODE>
__global__ void __launch_bounds__(512, 1) k_icache(unsigned long long* out, uint32_t* sink) {
  uint32_t a = threadIdx.x, b = blockIdx.x;
  unsigned long long c0, c1, c2;
  __syncthreads();
  c0 = clock64();
  for (int pass = 0; pass < 2; ++pass) {
    if (MODE == 0) { R1024(OPS) R1024(OPS) }           // 4096 instructions straight-line
    if (MODE == 1) { R64(OPS_SYNC) R64(OPS_SYNC) }      // 4096 instr + 128 barriers
    if (MODE == 2) { R256(OPS) }                         // 512 instructions
    __syncthreads();
    if (pass == 0) c1 = clock64();
  }
  c2 = clock64();
  if (threadIdx.x == 0) { out[blockIdx.x * 2] = c1 - c0; out[blockIdx.x * 2 + 1] = c2 - c1; }
  if (a == 0x12345 && b == 7) sink[0] = a;
}

template <int MODE>
int run(const char* name, int grid, int threads) {
  unsigned long long* out; uint32_t* sink;
  cudaMalloc(&out, grid * 16); cudaMalloc(&sink, 64);
  std::vector<unsigned long long> h(grid * 2);
  for (int rep = 0; rep < 3; ++rep) {
    k_icache<MODE><<<grid, threads>>>(out, sink);
    cudaDeviceSynchronize();
    cudaMemcpy(h.data(), out, grid * 16, cudaMemcpyDeviceToHost);
    std::vector<double> p1, p2;
    for (int i = 0; i < grid; ++i) { p1.push_back((double)h[2 * i]); p2.push_back((double)h[2 * i + 1]); }
    std::sort(p1.begin(), p1.end()); std::sort(p2.begin(), p2.end());
    printf("{\"probe\":\"icache\",\"mode\":\"%s\",\"grid\":%d,\"threads\":%d,\"rep\":%d,\"cold_pass_cyc_med\":%.0f,\"cold_max\":%.0f,\"warm_pass_cyc_med\":%.0f}\n",
           name, grid, threads, rep, p1[grid / 2], p1.back(), p2[grid / 2]);
  }
  cudaFree(out); cudaFree(sink);
  return 0;
}

int main() {
  run<0>("straight_4096", 144, 512);
  run<0>("straight_4096", 144, 32);
  run<1>("sync_every_32", 144, 512);
  run<2>("straight_512", 144, 512);
  return 0;
}
