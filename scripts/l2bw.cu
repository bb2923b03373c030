// L2 bandwidth microbenchmark (B200): each thread streams over an L2-resident
// working set of `ws` bytes (read-only, and read+write), 16-byte vector loads,
// grid = 148 SMs x 4 CTAs x 512 threads.  Prints GB/s per working-set size.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const double2* __restrict__ a, size_t n, int reps, double* out) {
  double s = 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
      double2 v = __ldcg(a + i);
      s += v.x + v.y;
    }
  if (s == 12345.678) *out = s;
}
__global__ void rw(double2* __restrict__ a, size_t n, int reps) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
      double2 v = __ldcg(a + i);
      v.x += 1.0;
      a[i] = v;
    }
}
int main() {
  double* out;
  cudaMalloc(&out, 8);
  for (size_t mb : {8, 16, 32, 48, 64, 96, 2048}) {
    size_t bytes = mb << 20, n = bytes / 16;
    double2* a;
    cudaMalloc(&a, bytes);
    cudaMemset(a, 0, bytes);
    int reps = mb >= 1024 ? 2 : (int)(4096 / mb);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    rd<<<148 * 4, 512>>>(a, n, 1, out);
    cudaEventRecord(e0);
    rd<<<148 * 4, 512>>>(a, n, reps, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double rdbw = (double)bytes * reps / (ms * 1e-3) / 1e9;
    rw<<<148 * 4, 512>>>(a, n, 1);
    cudaEventRecord(e0);
    rw<<<148 * 4, 512>>>(a, n, reps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double rwbw = 2.0 * bytes * reps / (ms * 1e-3) / 1e9;
    printf("ws %5zu MB  read %8.0f GB/s  read+write %8.0f GB/s\n", mb, rdbw, rwbw);
    cudaFree(a);
  }
  return 0;
}
