// Probe: dependent-chain latencies of the ops the selection phase uses
// (generic vs shared loads of smem data, VOTE, POPC) and a replica of the
// selection pass-1 row loop, 144 CTAs x 256 threads.  Not product code.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int MODE>
__global__ void __launch_bounds__(256, 1) k_chain(int iters, int* out, long long* cyc, int sel) {
  extern __shared__ __align__(16) uint32_t s[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = (i * 7 + 1) & 8191;
  __syncthreads();
  const uint32_t* gp = sel >= 0 ? s : nullptr;      // generic pointer to smem (opaque to the compiler)
  uint32_t v = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) v = s[v & 8191];                               // LDS chain
    if (MODE == 1) v = gp[v & 8191];                              // generic LD chain on smem
    if (MODE == 2) v = __ballot_sync(0xffffffffu, (v & 1) != 0) + v;  // VOTE chain
    if (MODE == 3) v = __popc(v) + v;                             // POPC chain
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = v;
}

// replica of selection pass 1: each warp scans SW tokens of a u16 D array in
// smem, rows of 64 tokens, 4 ballots per row, counts + a row list
template <bool GENERIC, int RU>
__global__ void __launch_bounds__(256, 1) k_pass1(int Lr, int thr, int* out, long long* cyc, int sel) {
  extern __shared__ __align__(16) uint32_t s[];
  uint16_t* D = reinterpret_cast<uint16_t*>(s);
  uint4* rmask = reinterpret_cast<uint4*>(s + 8192);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < Lr; i += blockDim.x) D[i] = (uint16_t)(200 + ((i * 2654435761u) >> 24) % 80);
  __syncthreads();
  const uint32_t* D32 = GENERIC ? (sel >= 0 ? reinterpret_cast<const uint32_t*>(D) : nullptr) : reinterpret_cast<const uint32_t*>(D);
  const int SW = (Lr + 8 * 64 - 1) / (8 * 64) * 64;
  const int w0 = min(Lr, warp * SW), w1 = min(Lr, w0 + SW);
  long long t0 = clock64();
  int lt = 0, ti = 0, nrl = 0;
  for (int jb = w0; jb < w1; jb += 64 * RU) {
    uint32_t m[RU][4];
#pragma unroll
    for (int q = 0; q < RU; ++q) {
      const int j = jb + 64 * q + 2 * lane;
      uint32_t v = 0xffffffffu;
      if (j < w1) v = D32[j >> 1];
      const int d0 = v & 0xffff, d1 = v >> 16;
      m[q][0] = __ballot_sync(0xffffffffu, d0 < thr);
      m[q][1] = __ballot_sync(0xffffffffu, d1 < thr);
      m[q][2] = __ballot_sync(0xffffffffu, d0 == thr);
      m[q][3] = __ballot_sync(0xffffffffu, d1 == thr);
    }
#pragma unroll
    for (int q = 0; q < RU; ++q) {
      lt += __popc(m[q][0]) + __popc(m[q][1]);
      ti += __popc(m[q][2]) + __popc(m[q][3]);
      if (m[q][0] | m[q][1] | m[q][2] | m[q][3]) {
        if (lane == 0 && nrl < 64) rmask[warp * 64 + nrl] = make_uint4(m[q][0], m[q][1], m[q][2], m[q][3]);
        ++nrl;
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = lt + ti + nrl;
}

// replica of the SWAR selection pass 1 (thread-contiguous 8-token blocks)
template <int VAR>
__global__ void __launch_bounds__(256, 1) k_swar(int Lr, int thr, int* out, long long* cyc, int sel) {
  extern __shared__ __align__(16) uint32_t s[];
  uint16_t* D = reinterpret_cast<uint16_t*>(s);
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) D[i] = i < Lr ? (uint16_t)(200 + ((i * 2654435761u) >> 24) % 80) : 0x7fff;
  __syncthreads();
  const int S8 = (Lr + 8 * 256 - 1) / (8 * 256);
  const uint4* Dv = (VAR == 1 && sel < 0 ? nullptr : reinterpret_cast<const uint4*>(D)) + threadIdx.x * S8;
  const uint32_t lt_k = (uint32_t)(thr - 1) * 0x10001u + 0x80008000u, le_k = (uint32_t)thr * 0x10001u + 0x80008000u;
  long long t0 = clock64();
  int lt = 0, eq = 0;
#pragma unroll 4
  for (int c = 0; c < S8; ++c) {
    const uint4 x = Dv[c];
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t l = (lt_k - w[q]) & 0x80008000u, e = ((le_k - w[q]) & 0x80008000u) & ~l;
      lt += __popc(l); eq += __popc(e);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = lt + 7 * eq;
}

int main() {
  int* io; long long* cyc; CK(cudaMalloc(&io, 148 * 1024 * 4)); CK(cudaMalloc(&cyc, 148 * 8));
  std::vector<long long> h(148);
  auto med = [&](int n) { std::vector<long long> v(h.begin(), h.begin() + n); std::sort(v.begin(), v.end()); return (double)v[n / 2]; };
  const int it = 4096;
  const int smem = 64 * 1024;
  cudaFuncSetAttribute(k_chain<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_chain<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_chain<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_chain<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* nm[] = {"lds", "generic_ld_smem", "vote", "popc"};
  for (int nt : {32, 256}) {
    k_chain<0><<<144, nt, smem>>>(it, io, cyc, 1); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h.data(), cyc, 144 * 8, cudaMemcpyDeviceToHost));
    printf("{\"probe\":\"chain\",\"op\":\"%s\",\"threads\":%d,\"cyc\":%.1f}\n", nm[0], nt, med(144) / it);
    k_chain<1><<<144, nt, smem>>>(it, io, cyc, 1); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h.data(), cyc, 144 * 8, cudaMemcpyDeviceToHost));
    printf("{\"probe\":\"chain\",\"op\":\"%s\",\"threads\":%d,\"cyc\":%.1f}\n", nm[1], nt, med(144) / it);
    k_chain<2><<<144, nt, smem>>>(it, io, cyc, 1); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h.data(), cyc, 144 * 8, cudaMemcpyDeviceToHost));
    printf("{\"probe\":\"chain\",\"op\":\"%s\",\"threads\":%d,\"cyc\":%.1f}\n", nm[2], nt, med(144) / it);
    k_chain<3><<<144, nt, smem>>>(it, io, cyc, 1); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h.data(), cyc, 144 * 8, cudaMemcpyDeviceToHost));
    printf("{\"probe\":\"chain\",\"op\":\"%s\",\"threads\":%d,\"cyc\":%.1f}\n", nm[3], nt, med(144) / it);
  }
  cudaFuncSetAttribute(k_pass1<true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_pass1<false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_pass1<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) {
    k_pass1<true, 4><<<144, 256, smem>>>(7296, 205, io, cyc, 1); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h.data(), cyc, 144 * 8, cudaMemcpyDeviceToHost));
    printf("{\"probe\":\"pass1\",\"generic\":1,\"RU\":4,\"cyc\":%.0f}\n", med(144));
    k_pass1<false, 4><<<144, 256, smem>>>(7296, 205, io, cyc, 1); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h.data(), cyc, 144 * 8, cudaMemcpyDeviceToHost));
    printf("{\"probe\":\"pass1\",\"generic\":0,\"RU\":4,\"cyc\":%.0f}\n", med(144));
    k_pass1<false, 1><<<144, 256, smem>>>(7296, 205, io, cyc, 1); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h.data(), cyc, 144 * 8, cudaMemcpyDeviceToHost));
    printf("{\"probe\":\"pass1\",\"generic\":0,\"RU\":1,\"cyc\":%.0f}\n", med(144));
  }
  cudaFuncSetAttribute(k_swar<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_swar<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) {
    k_swar<0><<<144, 256, smem>>>(7296, 205, io, cyc, 1); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h.data(), cyc, 144 * 8, cudaMemcpyDeviceToHost));
    printf("{\"probe\":\"swar\",\"var\":\"lds\",\"cyc\":%.0f}\n", med(144));
    k_swar<1><<<144, 256, smem>>>(7296, 205, io, cyc, 1); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h.data(), cyc, 144 * 8, cudaMemcpyDeviceToHost));
    printf("{\"probe\":\"swar\",\"var\":\"generic\",\"cyc\":%.0f}\n", med(144));
  }
  return 0;
}
