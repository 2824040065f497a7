// Development probe: HBM read bandwidth of the init pass's access pattern (32x32-int tiles of
// row-major planes, 128-byte row segments) versus contiguous streaming, on one B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void tiles(const int4* __restrict__ p, long long W4, long long H, long long planes, int* out) {
  // one CTA (256 threads) per 32x32 tile of each plane group of 10 planes; thread t: row t/8, 16 B
  const long long TX = W4 / 8, TY = H / 32;
  int acc = 0;
  for (long long tile = blockIdx.x; tile < TX * TY * (planes / 10); tile += gridDim.x) {
    const long long g = tile / (TX * TY), r = tile % (TX * TY), ty = r / TX, tx = r % TX;
    const int t = threadIdx.x;
    const long long y = ty * 32 + (t >> 3), x4 = tx * 8 + (t & 7);
#pragma unroll
    for (int pl = 0; pl < 10; ++pl) {
      const int4 v = __ldg(p + ((g * 10 + pl) * H + y) * W4 + x4);
      acc += v.x ^ v.y ^ v.z ^ v.w;
    }
  }
  if (acc == 0x12345) out[0] = acc;
}
__global__ void stream(const int4* __restrict__ p, long long n4, int* out) {
  int acc = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const int4 v = __ldg(p + i);
    acc += v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345) out[0] = acc;
}
int main() {
  const long long W = 1920, H = 1080, planes = 10 * 64;  // 64 frames of 10 planes
  const long long bytes = W * H * planes * 4;
  int4* p; int* out;
  cudaMalloc(&p, bytes); cudaMalloc(&out, 4);
  cudaMemset(p, 1, bytes);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int grid : {592, 1184, 2368, 4736}) {
    for (int rep = 0; rep < 2; ++rep) {
      float ms;
      cudaEventRecord(a); tiles<<<grid, 256>>>(p, W / 4, H - H % 32, planes, out); cudaEventRecord(b);
      cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
      const double tb = (double)(W * (H - H % 32) * planes * 4);
      if (rep) printf("tiles  grid %5d: %.2f ms  %.0f GB/s\n", grid, ms, tb / ms / 1e6);
      cudaEventRecord(a); stream<<<grid, 256>>>(p, bytes / 16, out); cudaEventRecord(b);
      cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("stream grid %5d: %.2f ms  %.0f GB/s\n", grid, ms, bytes / ms / 1e6);
    }
  }
  return 0;
}
