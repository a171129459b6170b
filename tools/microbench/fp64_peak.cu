// Calibration microbenchmark (not part of the product path).
// Measures on the B200 box:
//   * FP64 DFMA / DADD issue throughput (the second ceiling of the elasticity apply),
//   * a plain streaming copy / read / write with 8-B and 16-B accesses (HBM ceiling),
// so DESIGN.md can quote measured denominators next to MEASURED_PEAKS.json.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

template <int ILP>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double r[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) r[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) r[i] = fma(r[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += r[i];
  if (s == 123.456) out[0] = s;
}

template <int ILP>
__global__ void dadd_kernel(double* out, int iters, double a) {
  double r[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) r[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) r[i] = r[i] + a;
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += r[i];
  if (s == 123.456) out[0] = s;
}

__global__ void copy8(const double* __restrict__ a, double* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}
__global__ void copy16(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}
__global__ void read16(const double2* __restrict__ a, double* out, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t st = (size_t)gridDim.x * blockDim.x;
  double s = 0;
  for (; i < n; i += st) { double2 v = a[i]; s += v.x + v.y; }
  if (s == 123.456) out[0] = s;
}
__global__ void write16(double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = make_double2(1.0, 2.0);
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"clock_khz_attr\": %d}\n", p.name,
         p.multiProcessorCount, p.l2CacheSize, clk_khz);
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int sms = p.multiProcessorCount;
  // FP64 throughput: 8 warps/SM x 4 CTAs x ILP 8
  {
    const int iters = 20000;
    dim3 grid(sms * 4), block(256);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      dfma_kernel<8><<<grid, block>>>(out, iters, 0.999999, 1e-7);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)grid.x * block.x * iters * 8;
      printf("{\"test\": \"dfma\", \"rep\": %d, \"ms\": %.3f, \"Tinstr_per_s\": %.3f, \"per_sm_per_ns\": %.2f}\n",
             rep, ms, ops / ms / 1e9, ops / ms / 1e6 / sms);
    }
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      dadd_kernel<8><<<grid, block>>>(out, iters, 1e-7);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)grid.x * block.x * iters * 8;
      printf("{\"test\": \"dadd\", \"rep\": %d, \"ms\": %.3f, \"Tinstr_per_s\": %.3f}\n", rep, ms,
             ops / ms / 1e9);
    }
    // long run for clocks under sustained FP64 load (~2 s)
    cudaEventRecord(e0);
    for (int r = 0; r < 40; ++r) dfma_kernel<8><<<grid, block>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = 40.0 * grid.x * block.x * iters * 8;
    printf("{\"test\": \"dfma_sustained\", \"ms\": %.3f, \"Tinstr_per_s\": %.3f}\n", ms, ops / ms / 1e9);
  }
  // HBM
  {
    size_t n = (size_t)1 << 28;  // 2 GiB per buffer of doubles
    double *a, *b; CK(cudaMalloc(&a, n * 8)); CK(cudaMalloc(&b, n * 8));
    CK(cudaMemset(a, 0, n * 8)); CK(cudaMemset(b, 0, n * 8));
    for (int grid_mul : {4, 8, 16}) {
      dim3 grid(sms * grid_mul), block(256);
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0); copy8<<<grid, block>>>(a, b, n); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      printf("{\"test\": \"copy8\", \"grid_per_sm\": %d, \"GBps\": %.1f}\n", grid_mul, 2.0 * n * 8 / best / 1e6);
      best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0); copy16<<<grid, block>>>((double2*)a, (double2*)b, n / 2); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      printf("{\"test\": \"copy16\", \"grid_per_sm\": %d, \"GBps\": %.1f}\n", grid_mul, 2.0 * n * 8 / best / 1e6);
      best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0); read16<<<grid, block>>>((double2*)a, out, n / 2); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      printf("{\"test\": \"read16\", \"grid_per_sm\": %d, \"GBps\": %.1f}\n", grid_mul, 1.0 * n * 8 / best / 1e6);
      best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0); write16<<<grid, block>>>((double2*)b, n / 2); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      printf("{\"test\": \"write16\", \"grid_per_sm\": %d, \"GBps\": %.1f}\n", grid_mul, 1.0 * n * 8 / best / 1e6);
    }
  }
  return 0;
}
