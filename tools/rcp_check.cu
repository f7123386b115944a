// Accuracy of rcp_fast (shen_rows.cuh) against the correctly rounded 1/x over
// random doubles spanning many binades: max error in ulps and the seed's |e|.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1701_03787_b200/csrc -o /tmp/rc tools/rcp_check.cu && /tmp/rc
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "shen_rows.cuh"

__global__ void check(int64_t n, unsigned long long* maxulp, double* maxe, unsigned long long* nexact) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long worst = 0, exact = 0;
  double we = 0.0;
  for (; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = (uint64_t)i * 0x9E3779B97F4A7C15ull;
    h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 32;
    const double m = 1.0 + (double)(h >> 11) * 0x1.0p-53;       // [1, 2)
    const int ex = (int)(h % 1200) - 600;                       // 2^-600 .. 2^600
    const double x = ((h >> 7) & 1 ? -1.0 : 1.0) * scalbn(m, ex);
    const double r = shen::rcp_fast(x), ref = __drcp_rn(x);
    const long long d = llabs((long long)__double_as_longlong(r) - (long long)__double_as_longlong(ref));
    worst = d > (long long)worst ? d : worst;
    exact += d == 0;
    double r0;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r0) : "d"(x));
    we = fmax(we, fabs(__fma_rn(-x, r0, 1.0)));
  }
  atomicMax(maxulp, worst);
  atomicAdd(nexact, exact);
  atomicMax(reinterpret_cast<unsigned long long*>(maxe), (unsigned long long)__double_as_longlong(we));
}

int main() {
  const int64_t n = 1ll << 30;
  unsigned long long *mu, *ne;
  double* me;
  cudaMalloc(&mu, 8); cudaMalloc(&me, 8); cudaMalloc(&ne, 8);
  cudaMemset(mu, 0, 8); cudaMemset(me, 0, 8); cudaMemset(ne, 0, 8);
  check<<<148 * 8, 256>>>(n, mu, me, ne);
  unsigned long long hu, hn; double he;
  cudaMemcpy(&hu, mu, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&he, me, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(&hn, ne, 8, cudaMemcpyDeviceToHost);
  printf("rcp_fast over %lld doubles: max %llu ulp from 1/x, %.4f%% correctly rounded; seed max |e| = %.3e (2^%.1f)\n",
         (long long)n, hu, 100.0 * hn / n, he, log2(he));
  return cudaGetLastError() != cudaSuccess;
}
