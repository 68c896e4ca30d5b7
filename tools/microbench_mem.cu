// Ceilings of the memory access patterns the histogram count (K1) and the
// map kernel are bound by, measured on the B200 (run via gpurun; results in
// profiles/r02/microbench_mem.txt). Not part of the product.
//   * random RED pairs (RED.ADD count + RED.MAX ~index on one 8-B bin, the
//     K1 update) over a table of T bytes: pairs/s, for T = 32 MiB (one of
//     K1's four Morton-slice passes, L2-resident) and 128 MiB (the whole
//     table);
//   * random single-byte gathers from a 16 MiB table (the map's LUT): loads/s.
// Addresses come from a per-thread xorshift stream, so every access is an
// independent random bin (the cfg4 worst case: uniform 24-bit colors).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t xs(uint32_t& s) {
  s ^= s << 13;
  s ^= s >> 17;
  s ^= s << 5;
  return s;
}

__global__ void k_red_pairs(uint2* bins, uint32_t mask, int per_thread) {
  uint32_t s = 0x9E3779B9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  for (int i = 0; i < per_thread; ++i) {
    const uint32_t b = xs(s) & mask;
    uint32_t* p = reinterpret_cast<uint32_t*>(bins + b);
    atomicAdd(p, 1u);
    atomicMax(p + 1, ~(s & 0xFFFFFFu));
  }
}

__global__ void k_gather(const uint8_t* __restrict__ lut, uint32_t mask, int per_thread, uint32_t* out) {
  uint32_t s = 0x85EBCA6Bu * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  uint32_t acc = 0;
#pragma unroll 16
  for (int i = 0; i < per_thread; ++i) acc += __ldg(lut + (xs(s) & mask));
  if (acc == 0xFFFFFFFFu) out[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint2* bins;
  cudaMalloc(&bins, size_t(128) << 20);
  cudaMemset(bins, 0, size_t(128) << 20);
  uint8_t* lut;
  cudaMalloc(&lut, size_t(16) << 20);
  cudaMemset(lut, 1, size_t(16) << 20);
  uint32_t* out;
  cudaMalloc(&out, 64);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms = 0;
  const int threads = 256, per = 64;
  for (int mib : {32, 128}) {
    const uint32_t mask = (uint32_t)(((size_t)mib << 20) / 8 - 1);
    const int blocks = sms * 16;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      k_red_pairs<<<blocks, threads>>>(bins, mask, per);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(&ms, a, b);
    const double pairs = double(blocks) * threads * per;
    printf("random RED pairs (add + max on one 8-B bin) over %3d MiB: %.1f G pairs/s (%.1f G atomics/s)\n", mib,
           pairs / (ms * 1e-3) / 1e9, 2 * pairs / (ms * 1e-3) / 1e9);
  }
  {
    const uint32_t mask = (16u << 20) - 1;
    const int blocks = sms * 8;
    const int g = 256;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      k_gather<<<blocks, threads>>>(lut, mask, g, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(&ms, a, b);
    const double loads = double(blocks) * threads * g;
    printf("random 1-byte gathers from a 16 MiB table: %.1f G loads/s\n", loads / (ms * 1e-3) / 1e9);
  }
  const cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", e == cudaSuccess ? "no error" : cudaGetErrorString(e));
  return 0;
}
