// Calibration microbenchmark: cp.async.bulk (global -> shared) streaming throughput vs copy size.
// One producer warp per CTA streams `per_slot` copies of `bytes` each into an S-slot ring;
// one consumer warp waits (full) and releases (empty).  Reports achieved GB/s of HBM reads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_copy bulk_copy.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(d)), "l"(s), "r"(n), "r"(su32(b)) : "memory");
}

constexpr int S = 8;

__global__ void __launch_bounds__(64) stream(const char* src, size_t total, uint32_t bytes, int per_slot, int lanes) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)sm;
  uint64_t* empty = full + S;
  char* ring = (char*)(sm + 256);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t chunk = (size_t)bytes * per_slot;
  const size_t nchunks = total / chunk;
  int t = 0;
  if (warp == 0) {
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++t) {
      const int s = t & (S - 1);
      if (t >= S) mbar_wait(&empty[s], ((t / S) - 1) & 1);
      if (lane == 0) mbar_expect(&full[s], (uint32_t)chunk);
      __syncwarp();
      if (lane < lanes) for (int k = lane; k < per_slot; k += lanes)
        bulk(ring + (size_t)s * chunk + (size_t)k * bytes, src + c * chunk + (size_t)k * bytes, bytes, &full[s]);
    }
  } else {
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++t) {
      const int s = t & (S - 1);
      mbar_wait(&full[s], (t / S) & 1);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  size_t total = (size_t)2 << 30;
  char* src;
  cudaMalloc(&src, total);
  cudaMemset(src, 1, total);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  const uint32_t sizes[] = {128, 256, 512, 1024, 2048, 4096, 16384};
  for (int ctas_per_sm : {2, 4}) {
    for (uint32_t bytes : sizes) {
      for (int lanes : {1, 32}) {
        int per_slot = (int)((bytes >= 4096) ? 2 : (8192 / bytes));
        if (per_slot < 1) per_slot = 1;
        size_t smem = 256 + (size_t)S * bytes * per_slot;
        if (smem > 100000) { per_slot = (int)(90000 / S / bytes); if (per_slot < 1) continue; smem = 256 + (size_t)S * bytes * per_slot; }
        cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        float best = 1e9;
        for (int r = 0; r < 3; ++r) {
          cudaEventRecord(a);
          stream<<<sms * ctas_per_sm, 64, smem>>>(src, total, bytes, per_slot, lanes);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms; cudaEventElapsedTime(&ms, a, b);
          if (ms < best) best = ms;
        }
        cudaError_t e = cudaGetLastError();
        size_t moved = total / ((size_t)bytes * per_slot) * ((size_t)bytes * per_slot);
        printf("{\"ctas_per_sm\": %d, \"copy_bytes\": %u, \"copies_per_slot\": %d, \"issuing_lanes\": %d, \"GBps\": %.1f, \"copies_per_us_per_sm\": %.2f, \"err\": \"%s\"}\n",
               ctas_per_sm, bytes, per_slot, lanes, moved / best / 1e6, moved / (double)bytes / (best * 1e3) / sms, cudaGetErrorString(e));
      }
    }
  }
  return 0;
}
