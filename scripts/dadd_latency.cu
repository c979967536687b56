// Dev probe: dependent fp64 add-chain latency on the B200 (the floor of the
// strict long-row path). nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dadd scripts/dadd_latency.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(const double* v, int n, double* out, long long* cyc) {
  double acc = 0.0;
  long long t0 = clock64();
  #pragma unroll 16
  for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, v[i & 63]);
  long long t1 = clock64();
  out[0] = acc; cyc[0] = t1 - t0;
}
__global__ void chain_smem(int n, double* out, long long* cyc) {
  __shared__ double s[64];
  if (threadIdx.x < 64) s[threadIdx.x] = threadIdx.x * 0.5;
  __syncwarp();
  double acc = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < n; i += 64) {
    #pragma unroll
    for (int k = 0; k < 64; ++k) acc = __dadd_rn(acc, s[k]);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = acc; cyc[0] = t1 - t0; }
}
int main() {
  double *v, *o; long long* c; cudaMalloc(&v, 64*8); cudaMalloc(&o, 8); cudaMalloc(&c, 8);
  cudaMemset(v, 0, 512);
  int n = 1 << 20; long long h;
  chain<<<1,1>>>(v, n, o, c); cudaDeviceSynchronize();
  chain<<<1,1>>>(v, n, o, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("global-cached operand: %.2f cycles/add\n", double(h) / n);
  chain_smem<<<1,32>>>(n, o, c); cudaDeviceSynchronize();
  chain_smem<<<1,32>>>(n, o, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("smem operand (warp): %.2f cycles/add\n", double(h) / n);
  return 0;
}
