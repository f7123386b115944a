// DRAM efficiency of the access pattern a column-resident solve would use:
// persistent CTAs stream tiles of S consecutive systems x all rows of one
// parity of a (n_rows, B) complex128 array through shared memory with 2-D TMA
// boxes (S x 16 B wide, BLK rows tall) and write them back with TMA stores.
// Reports GB/s (read + write) per (S, BLK, slots).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tc tools/tile_copy.cu && /tmp/tc
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void mb_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(n));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(b)),
      "r"(phase) : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          (unsigned)__cvta_generic_to_shared(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void tma_store(const CUtensorMap* m, int c0, int c1, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(m), "r"(c0), "r"(c1),
               "r"((unsigned)__cvta_generic_to_shared(src)) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }

// tile t: systems [t*S, t*S+S), parity t & 1 (tensor maps 0/1), rows 0..np-1 in blocks of BLK
__global__ void tile_copy(const __grid_constant__ CUtensorMap in0, const __grid_constant__ CUtensorMap in1,
                          const __grid_constant__ CUtensorMap out0, const __grid_constant__ CUtensorMap out1,
                          int S, int BLK, int nslots, int np0, int np1, int64_t ntiles) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  unsigned char* slots = smem + 128;
  const unsigned blk_bytes = (unsigned)S * 16u * (unsigned)BLK;
  if (threadIdx.x == 0) {
    for (int k = 0; k < nslots; ++k) mb_init(bars + k, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  // flatten (tile, block) work items of this CTA
  int64_t t = blockIdx.x;
  int b = 0;
  struct Item { int64_t t; int b; };
  auto advance = [&](Item& it) {
    const int np = (it.t & 1) ? np1 : np0;
    const int nb = (np + BLK - 1) / BLK;
    if (++it.b == nb) { it.b = 0; it.t += gridDim.x; }
  };
  Item ld{t, b}, st{t, b};
  unsigned phase_bits = 0;
  int issued = 0;
  for (int k = 0; k < nslots && ld.t < ntiles; ++k) {
    const CUtensorMap* m = (ld.t & 1) ? &in1 : &in0;
    mb_expect(bars + k, blk_bytes);
    tma_load(slots + (size_t)k * blk_bytes, m, (int)((ld.t >> 1) * S * 2), ld.b * BLK, bars + k);
    advance(ld);
    ++issued;
  }
  int slot = 0;
  while (st.t < ntiles) {
    mb_wait(bars + slot, (phase_bits >> slot) & 1);
    phase_bits ^= 1u << slot;
    const CUtensorMap* mo = (st.t & 1) ? &out1 : &out0;
    tma_store(mo, (int)((st.t >> 1) * S * 2), st.b * BLK, slots + (size_t)slot * blk_bytes);
    advance(st);
    if (ld.t < ntiles) {
      bulk_wait_read<0>();
      const CUtensorMap* m = (ld.t & 1) ? &in1 : &in0;
      mb_expect(bars + slot, blk_bytes);
      tma_load(slots + (size_t)slot * blk_bytes, m, (int)((ld.t >> 1) * S * 2), ld.b * BLK, bars + slot);
      advance(ld);
    }
    slot = (slot + 1) % nslots;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int make_map(EncodeFn enc, CUtensorMap* m, double* base, int64_t B, int np, int S, int BLK) {
  cuuint64_t dims[2] = {(cuuint64_t)(2 * B), (cuuint64_t)np};
  cuuint64_t strides[1] = {(cuuint64_t)(2 * B * 16)};  // row stride of one parity: 2 rows
  cuuint32_t box[2] = {(cuuint32_t)(2 * S), (cuuint32_t)BLK};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r != CUDA_SUCCESS;
}

int main() {
  const int n_rows = 1023;
  const int64_t B = 2048LL * 1025;
  const int np0 = (n_rows + 1) / 2, np1 = n_rows / 2;
  double *in, *out;
  CK(cudaMalloc(&in, (size_t)n_rows * B * 16));
  CK(cudaMalloc(&out, (size_t)n_rows * B * 16));
  CK(cudaMemset(in, 0, (size_t)n_rows * B * 16));
  EncodeFn enc;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int Ss[] = {8, 16, 24, 32};
  const int BLKs[] = {32, 64, 128};
  for (int S : Ss)
    for (int BLK : BLKs) {
      const unsigned blk_bytes = S * 16 * BLK;
      const int nslots = std::min(32, (int)((200 * 1024) / blk_bytes));
      CUtensorMap m[4];
      if (make_map(enc, m + 0, in, B, np0, S, BLK) || make_map(enc, m + 1, in + 2 * B, B, np1, S, BLK) ||
          make_map(enc, m + 2, out, B, np0, S, BLK) || make_map(enc, m + 3, out + 2 * B, B, np1, S, BLK)) {
        printf("encode failed S=%d BLK=%d\n", S, BLK);
        continue;
      }
      const int64_t ntiles = 2 * ((B + S - 1) / S);
      const size_t smem = 128 + (size_t)nslots * blk_bytes;
      CK(cudaFuncSetAttribute(tile_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        tile_copy<<<sms, 32, smem>>>(m[0], m[1], m[2], m[3], S, BLK, nslots, np0, np1, ntiles);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep == 3)
          printf("S=%2d (%3d-B pieces) BLK=%3d slots=%2d (%3zu KB): %.2f ms  %.0f GB/s\n", S, S * 16, BLK, nslots,
                 smem / 1024, ms, 2.0 * n_rows * B * 16 / (ms * 1e6));
      }
    }
  CK(cudaGetLastError());
  return 0;
}
