// On-chip bandwidth peaks of this B200 for the roofline denominators of
// kernels that are not HBM-bound (the L2-resident persistent CG, the
// SM-resident CG): L2 read bandwidth over a 48 MB working set (L1 bypassed
// with ld.global.cg) and shared-memory bandwidth (64-bit loads, all SMs).
// Prints one JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o onchip_peaks onchip_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_l2_read(const double2* __restrict__ a, long long n, int reps, double* out) {
  double s0 = 0.0, s1 = 0.0;
  for (int r = 0; r < reps; ++r)
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
      const double2 v = __ldcg(a + i);
      s0 += v.x;
      s1 += v.y;
    }
  if (s0 + s1 == 1234.5) out[0] = s0;  // never true; keeps the loads
}

__device__ __forceinline__ double lds(const double* p) {  // volatile: never merged or hoisted
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}

__global__ void k_smem_read(int reps, double* out, long long* cyc) {
  extern __shared__ double sm[];
  const int n = 8192;  // 64 KB
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = i;
  __syncthreads();
  const long long c0 = clock64();
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int j = threadIdx.x;
  for (int r = 0; r < reps; ++r) {
    s0 += lds(sm + j);
    s1 += lds(sm + ((j + 1024) & (n - 1)));
    s2 += lds(sm + ((j + 2048) & (n - 1)));
    s3 += lds(sm + ((j + 3072) & (n - 1)));
    j = (j + 4096) & (n - 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - c0;
  if (s0 + s1 + s2 + s3 == 1234.5) out[0] = s0;
}

int main() {
  int nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // L2: 48 MB read repeatedly (resident after the first pass)
  const long long bytes = 48ll << 20, n = bytes / 16;
  double2* a;
  cudaMalloc(&a, bytes);
  cudaMemset(a, 0, bytes);
  const int reps = 40;
  k_l2_read<<<nsm * 4, 512>>>(a, n, 2, out);
  cudaEventRecord(e0);
  k_l2_read<<<nsm * 4, 512>>>(a, n, reps, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const double l2 = (double)bytes * reps / (ms * 1e-3) / 1e9;
  // shared memory: every SM, 1024 threads, 4 independent 8-byte loads per step
  const int sreps = 20000;
  cudaFuncSetAttribute(k_smem_read, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  long long* cyc;
  cudaMalloc(&cyc, nsm * sizeof(long long));
  k_smem_read<<<nsm, 1024, 65536>>>(100, out, cyc);
  cudaEventRecord(e0);
  k_smem_read<<<nsm, 1024, 65536>>>(sreps, out, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double sm = (double)nsm * 1024 * 4 * 8.0 * sreps / (ms * 1e-3) / 1e9;
  long long hc[1024];
  cudaMemcpy(hc, cyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
  double cmax = 0;
  for (int i = 0; i < nsm; ++i) cmax = hc[i] > cmax ? hc[i] : cmax;
  const double bpc = 1024.0 * 4 * 8.0 * sreps / cmax;  // bytes per SM clock (in-kernel clock64)
  printf("{\"_source\": \"tools/onchip_peaks.cu on one B200\", \"l2_gbs\": %.1f, "
         "\"smem_gbs\": %.1f, \"sm_count\": %d, \"clock_khz_attr\": %d, "
         "\"smem_bytes_per_clk_per_sm_at_attr_clock\": %.1f, \"smem_bytes_per_sm_clock64\": %.1f, "
         "\"smem_kernel_ms\": %.3f, \"err\": \"%s\"}\n",
         l2, sm, nsm, clk, sm * 1e9 / nsm / (clk * 1e3), bpc, ms,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
