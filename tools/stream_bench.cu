// Micro-benchmark: achievable HBM bandwidth of the CG sweep's access pattern
// (read p, r, x; write p, r, x; 8 B each per row) on B200.
//   1. contiguous grid-stride stream (the copy roofline for a 3-in/3-out mix)
//   2. warp column strips (32 lanes, 28 written), rows swept upwards, register
//      prefetch distance 3 -- the pattern of k_cg_iter's interior path
//   3. the same with a per-lane cp.async ring of depth 8
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bench stream_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void k_contig(const double* __restrict__ a, const double* __restrict__ b,
                         const double* __restrict__ c, double* __restrict__ d,
                         double* __restrict__ e, double* __restrict__ f, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double x = a[i], y = b[i], z = c[i];
    d[i] = x + 1.0;
    e[i] = y + 1.0;
    f[i] = z + 1.0;
  }
}

template <int KR>
__global__ void __launch_bounds__(128, 5) k_strips(const double* __restrict__ a,
                                                   const double* __restrict__ b,
                                                   const double* __restrict__ c,
                                                   double* __restrict__ d, double* __restrict__ e,
                                                   double* __restrict__ f, int w, int h,
                                                   int nstrips) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double s = 0;
  for (int blk = blockIdx.x; blk * 4 < nstrips * ((h + KR - 1) / KR); blk += gridDim.x) {
  const int task = blk * 4 + warp;
  const int rb = task / nstrips, strip = task % nstrips;
  int col = strip * 28 - 2 + lane;
  const bool out = lane >= 2 && lane < 30 && col < w;
  col = min(max(col, 0), w - 1);
  const int ly0 = rb * KR, ly1 = min(ly0 + KR, h);
  if (ly0 >= h) break;
  const double* pa = a + col;
  const double* pb = b + col;
  const double* pc = c + col;
  auto ld = [&](const double* p, int ly) { return ly < ly1 ? p[(long long)ly * w] : 0.0; };
  double a0 = ld(pa, ly0), b0 = ld(pb, ly0), c0 = ld(pc, ly0);
  double a1 = ld(pa, ly0 + 1), b1 = ld(pb, ly0 + 1), c1 = ld(pc, ly0 + 1);
  double a2 = ld(pa, ly0 + 2), b2 = ld(pb, ly0 + 2), c2 = ld(pc, ly0 + 2);
  for (int ly = ly0; ly < ly1; ++ly) {
    const double a3 = ld(pa, ly + 3), b3 = ld(pb, ly + 3), c3 = ld(pc, ly + 3);
    const double l = __shfl_up_sync(~0u, a0, 1), r = __shfl_down_sync(~0u, a0, 1);
    if (out) {
      const long long o = (long long)ly * w + col;
      d[o] = a0 + l + r;
      e[o] = b0 * 2.0;
      f[o] = c0 + 1.0;
    }
    s += b0;
    a0 = a1; b0 = b1; c0 = c1;
    a1 = a2; b1 = b2; c1 = c2;
    a2 = a3; b2 = b3; c2 = c3;
  }
  }
  if (s == 12345.0) d[0] = s;
}

__device__ __forceinline__ void cp8(double* s, const double* g) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(a), "l"(g) : "memory");
}

template <int KR, int D>
__global__ void __launch_bounds__(128, 5) k_strips_async(const double* __restrict__ a,
                                                         const double* __restrict__ b,
                                                         const double* __restrict__ c,
                                                         double* __restrict__ d,
                                                         double* __restrict__ e,
                                                         double* __restrict__ f, int w, int h,
                                                         int nstrips) {
  __shared__ double ring[4][D][3][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int task = blockIdx.x * 4 + warp;
  const int rb = task / nstrips, strip = task % nstrips;
  int col = strip * 28 - 2 + lane;
  const bool out = lane >= 2 && lane < 30 && col < w;
  col = min(max(col, 0), w - 1);
  const int ly0 = rb * KR, ly1 = min(ly0 + KR, h);
  if (ly0 >= h) return;
  auto issue = [&](int ly) {
    if (ly < ly1) {
      const long long o = (long long)ly * w + col;
      const int s = ly & (D - 1);
      cp8(&ring[warp][s][0][lane], a + o);
      cp8(&ring[warp][s][1][lane], b + o);
      cp8(&ring[warp][s][2][lane], c + o);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
#pragma unroll
  for (int i = 0; i < D - 1; ++i) issue(ly0 + i);
  double s = 0;
  for (int ly = ly0; ly < ly1; ++ly) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(D - 2) : "memory");
    const int sl = ly & (D - 1);
    const double a0 = ring[warp][sl][0][lane], b0 = ring[warp][sl][1][lane],
                 c0 = ring[warp][sl][2][lane];
    const double l = __shfl_up_sync(~0u, a0, 1), r = __shfl_down_sync(~0u, a0, 1);
    if (out) {
      const long long o = (long long)ly * w + col;
      d[o] = a0 + l + r;
      e[o] = b0 * 2.0;
      f[o] = c0 + 1.0;
    }
    s += b0;
    issue(ly + D - 1);
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  if (s == 12345.0) d[0] = s;
}

template <typename F>
float timeit(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  const int w = 768, h = 196608;
  const long long n = (long long)w * h;
  double* buf[6];
  for (auto& p : buf) {
    CK(cudaMalloc(&p, n * 8));
    CK(cudaMemset(p, 0, n * 8));
  }
  const double bytes = 6.0 * n * 8;
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float ms = timeit([&] { k_contig<<<nsm * 8, 256>>>(buf[0], buf[1], buf[2], buf[3], buf[4], buf[5], n); }, 10);
  printf("contiguous 3in/3out: %.3f ms %.0f GB/s\n", ms, bytes / ms / 1e6);
  const int nstrips = (w + 27) / 28;
  // strip pattern moves 28/32 of the written columns but reads the 4 halo lanes too
  const double sbytes = bytes;
#define RUN(KR)                                                                               \
  {                                                                                          \
    const int tasks = nstrips * ((h + KR - 1) / KR);                                         \
    float t = timeit([&] { k_strips<KR><<<(tasks + 3) / 4, 128>>>(buf[0], buf[1], buf[2],    \
                                                                  buf[3], buf[4], buf[5], w, \
                                                                  h, nstrips); }, 10);       \
    printf("strips regs krows=%d: %.3f ms %.0f GB/s\n", KR, t, sbytes / t / 1e6);           \
    t = timeit([&] { k_strips_async<KR, 8><<<(tasks + 3) / 4, 128>>>(                       \
                         buf[0], buf[1], buf[2], buf[3], buf[4], buf[5], w, h, nstrips); }, 10); \
    printf("strips async8 krows=%d: %.3f ms %.0f GB/s\n", KR, t, sbytes / t / 1e6);         \
    t = timeit([&] { k_strips_async<KR, 16><<<(tasks + 3) / 4, 128>>>(                      \
                         buf[0], buf[1], buf[2], buf[3], buf[4], buf[5], w, h, nstrips); }, 10); \
    printf("strips async16 krows=%d: %.3f ms %.0f GB/s\n", KR, t, sbytes / t / 1e6);        \
  }
  RUN(16) RUN(32) RUN(64) RUN(128)
  // occupancy sensitivity of the register version (dummy dynamic smem caps CTAs/SM)
  CK(cudaFuncSetAttribute(k_strips<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  for (int blocks : {2, 3, 4, 5, 6, 8, 10, 12, 16}) {
    const int tasks = nstrips * ((h + 31) / 32);
    float t = timeit([&] { k_strips<32><<<nsm * blocks, 128>>>(buf[0], buf[1], buf[2],
                                                                   buf[3], buf[4], buf[5], w, h,
                                                                   nstrips); }, 10);
    printf("strips regs krows=32 persistent grid %d x SM: %.3f ms %.0f GB/s\n", blocks, t, sbytes / t / 1e6);
  }
  for (int blocks : {3, 5, 9}) {
    const size_t sm = (size_t)(220 * 1024 / blocks) & ~size_t(1023);
    const int tasks = nstrips * ((h + 31) / 32);
    float t = timeit([&] { k_strips<32><<<(tasks + 3) / 4, 128, sm>>>(buf[0], buf[1], buf[2],
                                                                   buf[3], buf[4], buf[5], w, h,
                                                                   nstrips); }, 10);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_strips<32>, 128, sm);
    printf("strips regs krows=32 blocks/SM=%d: %.3f ms %.0f GB/s\n", occ, t, sbytes / t / 1e6);
  }
  CK(cudaGetLastError());
  return 0;
}
