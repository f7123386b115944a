// Access-pattern probe for a chunk-parallel streaming solve: does the second
// (backward) read of each row come from L2?  Each CTA takes a group of S
// consecutive systems x both parities x C chunks of K segments (8 rows each);
// thread = (system, parity, chunk).  Pass 1 reads the chunk's rows top-down
// (cp.async-free plain loads, accumulating), a CTA barrier, pass 2 re-reads
// them bottom-up and writes one complex per row.  Layout (rows, batch)
// complex128 like the solver's RHS.  Reports time; DRAM bytes come from ncu.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_reread tools/l2_reread.cu
#include <cstdio>
#include <cuda_runtime.h>

struct c2 { double x, y; };

template <int S, int C, int K>
__global__ void __launch_bounds__(S * 2 * C, 1) probe(const double2* __restrict__ rhs, double2* __restrict__ out,
                                                      int n_rows, long long B, long long ngroups) {
  const int tid = threadIdx.x;
  const int s = tid % S, rest = tid / S, par = rest & 1, c = rest >> 1;
  const int n = (n_rows - par + 1) / 2;
  const int rows_chunk = K * 8;
  for (long long g = blockIdx.x; g < ngroups; g += gridDim.x) {
    const long long j = g * S + s;
    double2 acc = make_double2(0.0, 0.0);
    const int i0 = c * rows_chunk, i1 = min(n, i0 + rows_chunk);
    for (int i = i0; i < i1; ++i) {
      const double2 v = __ldcg(rhs + (long long)(par + 2 * i) * B + j);
      acc.x = fma(acc.x, 0.5, v.x);
      acc.y = fma(acc.y, 0.5, v.y);
    }
    __syncthreads();
    for (int i = i1 - 1; i >= i0; --i) {
      const double2 v = __ldcg(rhs + (long long)(par + 2 * i) * B + j);
      acc.x = fma(acc.x, 0.5, v.x);
      acc.y = fma(acc.y, 0.5, v.y);
      __stcs(out + (long long)(par + 2 * i) * B + j, acc);
    }
    __syncthreads();
  }
}

template <int S, int C, int K>
void run(const double2* d_in, double2* d_out, int n_rows, long long B, int sms, int ctas) {
  const long long ngroups = B / S;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  probe<S, C, K><<<sms * ctas, S * 2 * C>>>(d_in, d_out, n_rows, B, ngroups);
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) probe<S, C, K><<<sms * ctas, S * 2 * C>>>(d_in, d_out, n_rows, B, ngroups);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 3;
  const double alg = 32.0 * n_rows * (double)B;
  printf("S=%2d C=%2d K=%d threads=%4d ctas/SM=%d: %.3f ms  alg %.0f GB/s (in-flight/SM %.0f KB)\n", S, C, K, S * 2 * C,
         ctas, ms, alg / ms / 1e6, ctas * S * 2.0 * C * K * 8 * 16 / 1024);
}

int main() {
  const int n_rows = 1023;           // config 4 Helmholtz modes
  const long long B = 2048LL * 1025; // config 4 systems
  double2 *d_in, *d_out;
  cudaMalloc(&d_in, sizeof(double2) * n_rows * B);
  cudaMalloc(&d_out, sizeof(double2) * n_rows * B);
  cudaMemset(d_in, 0, sizeof(double2) * n_rows * B);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<16, 16, 4>(d_in, d_out, n_rows, B, sms, 1);
  run<32, 8, 8>(d_in, d_out, n_rows, B, sms, 1);
  run<16, 8, 8>(d_in, d_out, n_rows, B, sms, 2);
  run<32, 16, 4>(d_in, d_out, n_rows, B, sms, 1);
  run<16, 32, 2>(d_in, d_out, n_rows, B, sms, 1);
  run<32, 4, 16>(d_in, d_out, n_rows, B, sms, 2);
  run<32, 2, 32>(d_in, d_out, n_rows, B, sms, 4);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
