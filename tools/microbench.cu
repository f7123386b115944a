// Dependent-chain latencies of the fp64 operations the solver recurrences
// are built from (one warp, clock64 around an unrolled chain).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench.cu && /tmp/mb
#include <cstdio>
#include <cuda_runtime.h>

#define N 512

__global__ void lat_kernel(double* out, long long* cyc, double a, double b) {
  double x = a + threadIdx.x * 1e-3;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) x = fma(x, b, a);
  t1 = clock64();
  cyc[0] = t1 - t0;
  out[0] = x;
  // DMUL chain
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) x = x * b;
  t1 = clock64();
  cyc[1] = t1 - t0;
  out[1] = x;
  // reciprocal (correctly rounded) chain
  x = 1.5 + threadIdx.x;
  t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) x = __drcp_rn(x) + 1.0;
  t1 = clock64();
  cyc[2] = t1 - t0;
  out[2] = x;
  // division chain
  x = 1.5 + threadIdx.x;
  t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) x = __ddiv_rn(a, x) + 1.0;
  t1 = clock64();
  cyc[3] = t1 - t0;
  out[3] = x;
  // approximate reciprocal: MUFU.RCP64H + 2 Newton steps, no slow path
  x = 1.5 + threadIdx.x;
  t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    x = r + 1.0;
  }
  t1 = clock64();
  cyc[4] = t1 - t0;
  out[4] = x;
}

__global__ void smem_lat_kernel(long long* cyc, int stride) {
  __shared__ unsigned idx[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) idx[i] = (i + stride) & 4095;
  __syncthreads();
  unsigned p = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) p = idx[p];
  long long t1 = clock64();
  cyc[5] = t1 - t0 + (p == 12345);
}

__global__ void thr_kernel(double* out, long long* cyc, double a, double b, int chains) {
  // throughput: 8 independent DFMA chains per thread, full SM of warps
  double x0 = a + threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
         x7 = x0 + 7;
  long long t0 = clock64();
  for (int i = 0; i < 1024; ++i) {
    x0 = fma(x0, b, a); x1 = fma(x1, b, a); x2 = fma(x2, b, a); x3 = fma(x3, b, a);
    x4 = fma(x4, b, a); x5 = fma(x5, b, a); x6 = fma(x6, b, a); x7 = fma(x7, b, a);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = t1 - t0;
  out[threadIdx.x + blockIdx.x * blockDim.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

int main() {
  double* d_out;
  long long* d_cyc;
  cudaMalloc(&d_out, 1 << 24);
  cudaMalloc(&d_cyc, 64 * sizeof(long long));
  lat_kernel<<<1, 32>>>(d_out, d_cyc, 0.5, 0.999);
  smem_lat_kernel<<<1, 32>>>(d_cyc, 33);
  long long c[8] = {0};
  cudaMemcpy(c, d_cyc, 6 * sizeof(long long), cudaMemcpyDeviceToHost);
  printf("latency (cycles per dependent op): DFMA %.1f  DMUL %.1f  drcp_rn+add %.1f  ddiv_rn+add %.1f  "
         "rcp.approx+2NR+add %.1f  LDS %.1f\n",
         c[0] / (double)N, c[1] / (double)N, c[2] / (double)N, c[3] / (double)N, c[4] / (double)N, c[5] / (double)N);
  for (int warps = 4; warps <= 32; warps *= 2) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    thr_kernel<<<148 * 4, warps * 8>>>(d_out, d_cyc, 0.5, 0.999, 8);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 1024 * 148 * 4 * warps * 8;
    printf("DFMA throughput, %d threads/block x 592 blocks: %.1f TFLOP/s\n", warps * 8, flops / ms / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
