// Does compute-sanitizer racecheck model mbarrier synchronisation?  A correct single-producer /
// single-consumer hand-off through shared memory guarded by two mbarriers (the pattern of the
// elasticity kernels' y hand-off and of the plane rings).  If racecheck reports hazards here, its
// reports on the apply kernels are tool false positives.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -o mbar_racecheck mbar_racecheck.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}\n"
               ::"r"(sa(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(sa(b)) : "memory");
}

__global__ void k(double* out, int rounds) {
  __shared__ double buf[4][32];
  __shared__ uint64_t full[4], empty[4];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x < 4) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sa(&full[threadIdx.x])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sa(&empty[threadIdx.x])));
  }
  __syncthreads();
  double acc = 0.0;
  for (int t = 0; t < rounds; ++t) {
    const int b = t & 3;
    const uint32_t n = t >> 2;
    if (w == 1) {  // producer
      if (n >= 1) wait(&empty[b], (n - 1) & 1);
      buf[b][lane] = t + lane;
      __syncwarp();
      if (lane == 0) arrive(&full[b]);
    } else {  // consumer
      wait(&full[b], n & 1);
      acc += buf[b][lane];
      __syncwarp();
      if (lane == 0) arrive(&empty[b]);
    }
  }
  if (w == 0) out[lane] = acc;
}

int main() {
  double* d;
  cudaMalloc(&d, 32 * sizeof(double));
  k<<<1, 64>>>(d, 64);
  double h[32];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double want = 0;
  for (int t = 0; t < 64; ++t) want += t;
  printf("{\"ok\": %s, \"lane0\": %g, \"want\": %g}\n", h[0] == want ? "true" : "false", h[0], want);
  return 0;
}
