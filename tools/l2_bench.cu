// Effective L2 capacity for the CG iteration's ping-pong pattern on B200:
// each launch reads K arrays of n doubles and writes K others, and the next
// launch reads what the previous one wrote.  Time per launch vs footprint
// shows where the working set stops being L2-resident.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_bench l2_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_pingpong(const double* __restrict__ a, const double* __restrict__ b,
                           const double* __restrict__ c, double* __restrict__ d,
                           double* __restrict__ e, double* __restrict__ f, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    d[i] = a[i] + 1.0;
    e[i] = b[i] + 1.0;
    f[i] = c[i] + 1.0;
  }
}

// x updated in place + r, p double buffered (the CG layout)
__global__ void k_cg_like(double* __restrict__ x, const double* __restrict__ r0,
                          const double* __restrict__ p0, double* __restrict__ r1,
                          double* __restrict__ p1, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double p = p0[i];
    x[i] += 0.5 * p;
    r1[i] = r0[i] - p;
    p1[i] = p * 0.25 + r0[i];
  }
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const long long nmax = 64ll << 20 >> 3;  // 64 MiB per array
  double* buf[6];
  for (auto& p : buf) {
    cudaMalloc(&p, nmax * 8);
    cudaMemset(p, 0, nmax * 8);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mb : {2, 4, 6, 8, 10, 12, 14, 16, 20, 24, 32, 48, 64}) {
    const long long n = (long long)mb << 20 >> 3;
    const int reps = 50;
    for (int variant = 0; variant < 2; ++variant) {
      auto launch = [&](int it) {
        if (variant == 0) {
          if (it & 1)
            k_pingpong<<<nsm * 8, 256>>>(buf[3], buf[4], buf[5], buf[0], buf[1], buf[2], n);
          else
            k_pingpong<<<nsm * 8, 256>>>(buf[0], buf[1], buf[2], buf[3], buf[4], buf[5], n);
        } else {
          if (it & 1)
            k_cg_like<<<nsm * 8, 256>>>(buf[0], buf[3], buf[4], buf[1], buf[2], n);
          else
            k_cg_like<<<nsm * 8, 256>>>(buf[0], buf[1], buf[2], buf[3], buf[4], n);
        }
      };
      for (int it = 0; it < 4; ++it) launch(it);
      cudaEventRecord(e0);
      for (int it = 0; it < reps; ++it) launch(it);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double us = ms * 1e3 / reps;
      const double bytes = variant == 0 ? 6.0 * n * 8 : 6.0 * n * 8;  // 3 in + 3 out
      const double foot = variant == 0 ? 6.0 * mb : 5.0 * mb;
      printf("%s %3d MiB/array footprint %4.0f MiB: %8.2f us/launch %7.0f GB/s\n",
             variant == 0 ? "pingpong" : "cg_like ", mb, foot, us, bytes / us / 1e3);
    }
  }
  return 0;
}
