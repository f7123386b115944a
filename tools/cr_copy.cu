// DRAM efficiency of the column-resident (CR) solve's data movement, with the
// compute stubbed: persistent CTAs of NT threads walk tiles of S consecutive
// systems x all rows of one parity of a (n_rows, B) complex128 array; each
// tile is loaded by 2-D TMA boxes (S x 16 B wide, BOX rows tall, parity
// stride 2 rows) into one of NSLOT shared-memory slots, every thread then
// reads and rewrites its chunk (a contiguous run of rows of one system, the
// CR kernels' smem access pattern), and the tile is written back by TMA.
// Reports GB/s (read + write).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/crc tools/cr_copy.cu && /tmp/crc
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstring>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, unsigned phase) {
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(su32(b)),
               "r"(phase) : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          su32(dst)), "l"(m), "r"(c0), "r"(c1), "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void tma_store(const CUtensorMap* m, int c0, int c1, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(m), "r"(c0), "r"(c1),
               "r"(su32(src)) : "memory");
}

template <int S, int NSLOT, int NT, int BOX>
__global__ void __launch_bounds__(NT, 1) cr_copy(const __grid_constant__ CUtensorMap in0, const __grid_constant__ CUtensorMap in1,
                                               const __grid_constant__ CUtensorMap out0, const __grid_constant__ CUtensorMap out1,
                                               int np0, int np1, int64_t ntiles) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  constexpr int ROWB = S * 16;
  const int npmax = np0;
  const size_t slot_bytes = (size_t)npmax * ROWB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NSLOT * slot_bytes);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int k = 0; k < NSLOT; ++k) mb_init(bars + k, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue_load = [&](int64_t t, int slot) {
    const int par = (int)(t & 1), np = par ? np1 : np0;
    const CUtensorMap* m = par ? &in1 : &in0;
    mb_expect(bars + slot, (unsigned)(((np + BOX - 1) / BOX) * BOX * ROWB));  // full boxes (OOB rows zero-filled)
    for (int r = 0; r < np; r += BOX) tma_load(smem + slot * slot_bytes + (size_t)r * ROWB, m, (int)((t >> 1) * S * 2), r, bars + slot);
  };
  int64_t t_ld = blockIdx.x;
  // prologue: fill all but one slot
  if (tid == 0)
    for (int k = 0; k < NSLOT - 1 && t_ld < ntiles; ++k, t_ld += gridDim.x) issue_load(t_ld, k);
  unsigned phase = 0;
  int slot = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int par = (int)(t & 1), np = par ? np1 : np0;
    // refill the slot that was stored last iteration (its store must have been read out)
    if (tid == 0 && t_ld < ntiles) {
      const int ls = (slot + NSLOT - 1) % NSLOT;
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      issue_load(t_ld, ls);
      t_ld += gridDim.x;
    }
    mb_wait(bars + slot, (phase >> slot) & 1);
    phase ^= 1u << slot;
    // "compute": thread = (system s, chunk c) over contiguous row runs
    double2* tile = reinterpret_cast<double2*>(smem + slot * slot_bytes);
    constexpr int NCH = NT / S;
    const int s = tid % S, c = tid / S;
    const int rpc = (np + NCH - 1) / NCH;
    for (int r = c * rpc; r < min(np, (c + 1) * rpc); ++r) {
      double2 v = tile[r * S + s];
      v.x += 1.0;
      tile[r * S + s] = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      const CUtensorMap* m = par ? &out1 : &out0;
      for (int r = 0; r < np; r += BOX) tma_store(m, (int)((t >> 1) * S * 2), r, smem + slot * slot_bytes + (size_t)r * ROWB);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    slot = (slot + 1) % NSLOT;
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Row-blocked tiles (the cluster variant's per-CTA share): tile t = (system
// block sb, parity, row block rb of RB rows); consecutive t are the row blocks
// of one (sb, parity), i.e. the CTAs of one cluster run side by side.
template <int S, int NSLOT, int NT, int RB>
__global__ void __launch_bounds__(NT, 1) cr_copy_rb(const __grid_constant__ CUtensorMap in0, const __grid_constant__ CUtensorMap in1,
                                                  const __grid_constant__ CUtensorMap out0, const __grid_constant__ CUtensorMap out1,
                                                  int np0, int np1, int64_t ntiles, int nrb) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  constexpr int ROWB = S * 16;
  const size_t slot_bytes = (size_t)RB * ROWB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NSLOT * slot_bytes);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int k = 0; k < NSLOT; ++k) mb_init(bars + k, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto coords = [&](int64_t t, int& par, int& c0, int& r0) {
    const int64_t sb = t / (2 * nrb);
    par = (int)((t / nrb) & 1);
    r0 = (int)(t % nrb) * RB;
    c0 = (int)(sb * S * 2);
  };
  auto issue_load = [&](int64_t t, int slot) {
    int par, c0, r0;
    coords(t, par, c0, r0);
    mb_expect(bars + slot, (unsigned)(RB * ROWB));
    tma_load(smem + slot * slot_bytes, par ? &in1 : &in0, c0, r0, bars + slot);
  };
  int64_t t_ld = blockIdx.x;
  if (tid == 0)
    for (int k = 0; k < NSLOT - 1 && t_ld < ntiles; ++k, t_ld += gridDim.x) issue_load(t_ld, k);
  unsigned phase = 0;
  int slot = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    if (tid == 0 && t_ld < ntiles) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      issue_load(t_ld, (slot + NSLOT - 1) % NSLOT);
      t_ld += gridDim.x;
    }
    mb_wait(bars + slot, (phase >> slot) & 1);
    phase ^= 1u << slot;
    double2* tile = reinterpret_cast<double2*>(smem + slot * slot_bytes);
    constexpr int NCH = NT / S;
    const int s = tid % S, c = tid / S;
    constexpr int rpc = (RB + NCH - 1) / NCH;
    for (int r = c * rpc; r < min(RB, (c + 1) * rpc); ++r) {
      double2 v = tile[r * S + s];
      v.x += 1.0;
      tile[r * S + s] = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      int par, c0, r0;
      coords(t, par, c0, r0);
      tma_store(par ? &out1 : &out0, c0, r0, smem + slot * slot_bytes);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    slot = (slot + 1) % NSLOT;
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static int make_map(EncodeFn enc, CUtensorMap* m, double* base, int64_t B, int np, int S, int BOX, CUtensorMapL2promotion pr) {
  cuuint64_t dims[2] = {(cuuint64_t)(2 * B), (cuuint64_t)np};
  cuuint64_t strides[1] = {(cuuint64_t)(2 * B * 16)};
  cuuint32_t box[2] = {(cuuint32_t)(2 * S), (cuuint32_t)BOX};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS;
}

template <int S, int NSLOT, int NT, int BOX>
static int run(EncodeFn enc, double* in, double* out, int n_rows, int64_t B, int sms, int ctas_per_sm, CUtensorMapL2promotion pr,
               const char* prn) {
  const int np0 = (n_rows + 1) / 2, np1 = n_rows / 2;
  CUtensorMap m[4];
  if (make_map(enc, m + 0, in, B, np0, S, BOX, pr) || make_map(enc, m + 1, in + 2 * B, B, np1, S, BOX, pr) ||
      make_map(enc, m + 2, out, B, np0, S, BOX, pr) || make_map(enc, m + 3, out + 2 * B, B, np1, S, BOX, pr)) {
    printf("encode failed\n");
    return 1;
  }
  const size_t smem = (size_t)NSLOT * np0 * S * 16 + 64 + 1024;
  auto k = cr_copy<S, NSLOT, NT, BOX>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t ntiles = 2 * (B / S);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    k<<<sms * ctas_per_sm, NT, smem>>>(m[0], m[1], m[2], m[3], np0, np1, ntiles);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  printf("S=%2d NSLOT=%d NT=%3d BOX=%3d ctas/SM=%d promo=%s smem=%3zu KB: %.2f ms  %.0f GB/s\n", S, NSLOT, NT, BOX,
         ctas_per_sm, prn, smem / 1024, best, 2.0 * n_rows * (double)(B / S * S) * 16 / (best * 1e6));
  fflush(stdout);
  return 0;
}

template <int S, int NSLOT, int NT, int RB>
static int run_rb(EncodeFn enc, double* in, double* out, int n_rows, int64_t B, int sms) {
  const int np0 = (n_rows + 1) / 2, np1 = n_rows / 2;
  const auto pr = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  CUtensorMap m[4];
  if (make_map(enc, m + 0, in, B, np0, S, RB, pr) || make_map(enc, m + 1, in + 2 * B, B, np1, S, RB, pr) ||
      make_map(enc, m + 2, out, B, np0, S, RB, pr) || make_map(enc, m + 3, out + 2 * B, B, np1, S, RB, pr)) {
    printf("encode failed\n");
    return 1;
  }
  const int nrb = (np0 + RB - 1) / RB;
  const size_t smem = (size_t)NSLOT * RB * S * 16 + 64 + 1024;
  auto k = cr_copy_rb<S, NSLOT, NT, RB>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t ntiles = 2 * (B / S) * nrb;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    k<<<sms, NT, smem>>>(m[0], m[1], m[2], m[3], np0, np1, ntiles, nrb);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  printf("rowblock S=%2d RB=%3d NSLOT=%d NT=%3d smem=%3zu KB: %.2f ms  %.0f GB/s\n", S, RB, NSLOT, NT, smem / 1024, best,
         2.0 * n_rows * (double)(B / S * S) * 16 / (best * 1e6));
  fflush(stdout);
  return 0;
}

int main() {
  const int n_rows = 1023;
  const int64_t B = 2048LL * 1025;
  double *in, *out;
  CK(cudaMalloc(&in, (size_t)n_rows * B * 16));
  CK(cudaMalloc(&out, (size_t)n_rows * B * 16));
  CK(cudaMemset(in, 0, (size_t)n_rows * B * 16));
  EncodeFn enc;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const auto P2 = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  run<16, 1, 512, 256>(enc, in, out, n_rows, B, sms, 1, P2, "256B");
  run_rb<16, 3, 256, 256>(enc, in, out, n_rows, B, sms);
  run_rb<16, 3, 256, 128>(enc, in, out, n_rows, B, sms);
  run_rb<16, 6, 256, 128>(enc, in, out, n_rows, B, sms);
  run_rb<32, 3, 256, 128>(enc, in, out, n_rows, B, sms);
  run_rb<32, 6, 256, 64>(enc, in, out, n_rows, B, sms);
  run_rb<32, 3, 256, 64>(enc, in, out, n_rows, B, sms);
  run_rb<64, 3, 256, 64>(enc, in, out, n_rows, B, sms);
  run_rb<16, 12, 256, 64>(enc, in, out, n_rows, B, sms);
  return 0;
}
