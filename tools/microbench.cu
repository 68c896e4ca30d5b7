// Microbenchmarks of the primitives the WSM loop is built from (run on the
// B200 via gpurun; results recorded in profiles/). Not part of the product.
//   FP64 / FP32 / INT dependent-chain latency, FP64 throughput,
//   cooperative grid.sync cost vs a hand-rolled barrier, LDS latency.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__global__ void k_lat_dadd(double* out, int n, double a) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, a);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) out[1000] = double(t1 - t0) / n;
}
__global__ void k_lat_dmul(double* out, int n, double a) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dmul_rn(x, a);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) out[1000] = double(t1 - t0) / n;
}
__global__ void k_lat_fadd(float* out, int n, float a) {
  float x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __fadd_rn(x, a);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) out[1000] = float(t1 - t0) / n;
}
// throughput: 8 independent chains per thread, many warps
__global__ void k_tput_dfma(double* out, int n, double a) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < n; ++i) {
    x0 = __dadd_rn(x0, a); x1 = __dadd_rn(x1, a); x2 = __dadd_rn(x2, a); x3 = __dadd_rn(x3, a);
    x4 = __dadd_rn(x4, a); x5 = __dadd_rn(x5, a); x6 = __dadd_rn(x6, a); x7 = __dadd_rn(x7, a);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void k_tput_fadd(float* out, int n, float a) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < n; ++i) {
    x0 = __fadd_rn(x0, a); x1 = __fadd_rn(x1, a); x2 = __fadd_rn(x2, a); x3 = __fadd_rn(x3, a);
    x4 = __fadd_rn(x4, a); x5 = __fadd_rn(x5, a); x6 = __fadd_rn(x6, a); x7 = __fadd_rn(x7, a);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void k_lat_lds(int* out, int n) {
  __shared__ int s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i + 1) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) p = s[p];
  long long t1 = clock64();
  out[threadIdx.x] = p;
  if (threadIdx.x == 0) out[1000] = int((t1 - t0) / n);
}

__global__ void k_gridsync(long long* out, int n) {
  cg::grid_group g = cg::this_grid();
  long long t0 = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < n; ++i) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    out[0] = (t1 - t0) / n;
  }
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Sense-free barrier on a monotonically increasing arrival counter.
__device__ __forceinline__ void bar_grid(unsigned* ctr, unsigned& epoch) {
  __syncthreads();
  epoch += gridDim.x;
  if (threadIdx.x == 0) {
    red_release(ctr, 1u);
    while ((int)(ld_acquire(ctr) - epoch) < 0) {
    }
  }
  __syncthreads();
}
__global__ void k_mybar(long long* out, unsigned* ctr, int n) {
  unsigned epoch = 0;
  long long t0 = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < n; ++i) bar_grid(ctr, epoch);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    out[0] = (t1 - t0) / n;
  }
}

int main() {
  double* dd;
  float* df;
  int* di;
  long long* dl;
  unsigned* dc;
  cudaMalloc(&dd, 1 << 24);
  cudaMalloc(&df, 1 << 24);
  cudaMalloc(&di, 1 << 20);
  cudaMalloc(&dl, 64);
  cudaMalloc(&dc, 64);
  double h;
  float hf;
  int hi;
  long long hl;
  k_lat_dadd<<<1, 32>>>(dd, 4096, 1.0000001);
  cudaMemcpy(&h, dd + 1000, 8, cudaMemcpyDeviceToHost);
  printf("DADD dependent latency: %.1f cycles\n", h);
  k_lat_dmul<<<1, 32>>>(dd, 4096, 1.0000001);
  cudaMemcpy(&h, dd + 1000, 8, cudaMemcpyDeviceToHost);
  printf("DMUL dependent latency: %.1f cycles\n", h);
  k_lat_fadd<<<1, 32>>>(df, 4096, 1.0000001f);
  cudaMemcpy(&hf, df + 1000, 4, cudaMemcpyDeviceToHost);
  printf("FADD dependent latency: %.1f cycles\n", hf);
  k_lat_lds<<<1, 32>>>(di, 4096);
  cudaMemcpy(&hi, di + 1000, 4, cudaMemcpyDeviceToHost);
  printf("LDS dependent latency: %d cycles\n", hi);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int n = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    k_tput_dfma<<<sms * 4, 512>>>(dd, n, 1.0000001);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("DADD throughput: %.2f T ops/s (%.1f per SM per clk at 1.965 GHz)\n",
         double(sms) * 4 * 512 * n * 8 / (ms * 1e-3) / 1e12, double(sms) * 4 * 512 * n * 8 / (ms * 1e-3) / sms / 1.965e9);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    k_tput_fadd<<<sms * 4, 512>>>(df, n, 1.0000001f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  cudaEventElapsedTime(&ms, a, b);
  printf("FADD throughput: %.2f T ops/s (%.1f per SM per clk)\n",
         double(sms) * 4 * 512 * n * 8 / (ms * 1e-3) / 1e12, double(sms) * 4 * 512 * n * 8 / (ms * 1e-3) / sms / 1.965e9);
  for (int bpsm : {1, 2}) {
    for (int threads : {256, 512, 1024}) {
      if (threads * bpsm > 2048) continue;
      int nb = sms * bpsm;
      int iters = 2000;
      void* args[] = {&dl, &iters};
      cudaLaunchCooperativeKernel((void*)k_gridsync, nb, threads, args, 0, 0);
      cudaMemcpy(&hl, dl, 8, cudaMemcpyDeviceToHost);
      printf("cg grid.sync  blocks=%4d threads=%4d : %lld ns\n", nb, threads, hl);
      cudaMemset(dc, 0, 64);
      void* args2[] = {&dl, &dc, &iters};
      cudaLaunchCooperativeKernel((void*)k_mybar, nb, threads, args2, 0, 0);
      cudaMemcpy(&hl, dl, 8, cudaMemcpyDeviceToHost);
      printf("red/acquire bar blocks=%4d threads=%4d : %lld ns\n", nb, threads, hl);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
