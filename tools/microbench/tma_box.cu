// Calibration microbenchmark: TMA tensor box loads (cp.async.bulk.tensor.3d) streaming
// throughput vs box shape (W doubles x H rows per plane).  One producer lane per CTA streams the
// planes of its xy tile through an S-slot ring; one consumer warp waits and releases.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_box tma_box.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

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
__device__ __forceinline__ void tma3(void* d, const CUtensorMap* m, int x, int y, int z, uint64_t* b) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(su32(d)), "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(z), "r"(su32(b)) : "memory");
}

constexpr int S = 8;

__global__ void __launch_bounds__(64) stream(const __grid_constant__ CUtensorMap map, int W, int H, int nz, int tiles_x) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)sm;
  uint64_t* empty = full + S;
  unsigned char* ring = sm + 1024;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int bytes = W * H * 8;
  const int slot_bytes = (bytes + 127) & ~127;
  const int x0 = (blockIdx.x % tiles_x) * W, y0 = (blockIdx.x / tiles_x) * H;
  if (warp == 0) {
    if (lane == 0)
      for (int t = 0; t < nz; ++t) {
        const int s = t & (S - 1);
        if (t >= S) mbar_wait(&empty[s], ((t / S) - 1) & 1);
        mbar_expect(&full[s], bytes);
        tma3(ring + s * slot_bytes, &map, x0, y0, t, &full[s]);
      }
  } else {
    for (int t = 0; t < nz; ++t) {
      const int s = t & (S - 1);
      mbar_wait(&full[s], (t / S) & 1);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  const int NX = 2048, NY = 1024, NZ = 96;  // doubles: 1.6 GB
  double* buf;
  cudaMalloc(&buf, (size_t)NX * NY * NZ * 8);
  cudaMemset(buf, 0, (size_t)NX * NY * NZ * 8);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  const int shapes[][2] = {{36, 18}, {102, 10}, {102, 16}, {64, 16}, {128, 8}, {128, 16}, {256, 8}, {256, 4}, {256, 16}, {32, 32}};
  for (auto& sh : shapes) {
    const int W = sh[0], H = sh[1];
    CUtensorMap m;
    cuuint64_t dims[3] = {NX, NY, NZ};
    cuuint64_t str[2] = {NX * 8ull, (cuuint64_t)NX * NY * 8ull};
    cuuint32_t box[3] = {(cuuint32_t)W, (cuuint32_t)H, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int tiles_x = NX / W, tiles_y = NY / H;
    const int grid = tiles_x * tiles_y;
    const int slot_bytes = (W * H * 8 + 127) & ~127;
    const size_t smem = 1024 + (size_t)S * slot_bytes;
    cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    float best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      stream<<<grid, 64, smem>>>(m, W, H, NZ, tiles_x);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    const double bytes = (double)tiles_x * W * tiles_y * H * NZ * 8;
    const double rows = (double)grid * NZ * H;
    printf("{\"W\": %d, \"H\": %d, \"encode\": %d, \"GBps\": %.1f, \"rows_per_us_per_sm\": %.1f, \"boxes_per_us_per_sm\": %.2f, \"grid\": %d, \"err\": \"%s\"}\n",
           W, H, (int)r, bytes / best / 1e6, rows / (best * 1e3) / sms, grid * (double)NZ / (best * 1e3) / sms, grid,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
