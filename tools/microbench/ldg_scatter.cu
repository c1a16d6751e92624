// Microbenchmark: cost of the judge's scattered per-lane row loads (every
// lane streams its own far-away run) as 128-bit vs 256-bit loads, alone and
// mixed with the per-event shared atomic + u16 load/store traffic of the
// hot loop.  192 threads, one CTA per SM (the judge's shape).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s line %d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__device__ __forceinline__ uint32_t hsh(uint32_t x){ x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x; }

__device__ __forceinline__ void ld4(const uint16_t* p, uint32_t (&r)[8], int o) {
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r[o]),"=r"(r[o+1]),"=r"(r[o+2]),"=r"(r[o+3]) : "l"(p));
}
__device__ __forceinline__ void ld8(const uint16_t* p, uint32_t (&r)[8]) {
  asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]) : "l"(p));
}

// V8: 0 = two 128-bit loads per 32 B, 1 = one 256-bit load.  EV: events per 16 pixels of
// 3 rows (0 = loads only).
template <int V8, int EV, int T = 192>
__global__ void __launch_bounds__(T, 1) k(const uint16_t* __restrict__ img, int64_t npix, int W, int steps, uint32_t* out) {
  extern __shared__ uint32_t h[];
  for (int i = threadIdx.x; i < 32768 + 12 * 64 * 32; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int lanes = gridDim.x * blockDim.x;
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  int64_t run = (npix / lanes) & ~int64_t(15);
  int64_t a = g * run;
  uint32_t acc = 0, st = hsh(g);
  uint8_t* lt = reinterpret_cast<uint8_t*>(h + 32768) + (threadIdx.x & 31) * 4 + ((threadIdx.x >> 5) % 12) * 64 * 128;
  for (int s = 0; s < steps; ++s) {
    int64_t p = a + (int64_t)(s * 16) % run;
    uint32_t r[3][8];
    for (int row = 0; row < 3; ++row) {
      int64_t o = p - (int64_t)(row == 0 ? 0 : row == 1 ? W : 15 * W);
      if (o < 0) o += npix;
      if (V8) ld8(img + o, r[row]);
      else { ld4(img + o, r[row], 0); ld4(img + o + 8, r[row], 4); }
    }
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) x ^= r[0][i] + r[1][i] * 3 + r[2][i] * 5;
    acc ^= x;
    if (EV) {
#pragma unroll
      for (int e = 0; e < EV; ++e) {
        uint32_t key = (x >> (e & 15)) & 255;
        uint32_t la = (key & 63) * 128 + (key >> 6);
        uint32_t last = lt[la];
        lt[la] = (uint8_t)(x + e);
        uint32_t w = (last * 131 + hsh(st + e)) & 32767;
        acc += atomicAdd(&h[w], 1u);
      }
      st += 0x9e3779b9u;
    }
  }
  if (acc == 0x12345678) out[0] = acc;
}

template <int V8, int EV, int T = 192>
int run(const uint16_t* img, int64_t npix, int W, int nsm, uint32_t* out, const char* name) {
  int smem = 32768 * 4 + 12 * 64 * 128;
  CK(cudaFuncSetAttribute(k<V8, EV, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int steps = 20000;
  k<V8, EV, T><<<nsm, T, smem>>>(img, npix, W, 200, out);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<V8, EV, T><<<nsm, T, smem>>>(img, npix, W, steps, out);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double clk = 1.965e9 * ms * 1e-3;
  double lanepix = (double)nsm * T * steps * 16;
  printf("%-22s %8.3f ms  %.3f lane-pixels/clk/SM  %.3f events/clk/SM\n", name, ms, lanepix / clk / nsm,
         EV ? lanepix / 16 * EV / clk / nsm : 0.0);
  return 0;
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int W = 2048; const int64_t npix = 16LL * 2048 * 2048;
  uint16_t* img; uint32_t* out;
  CK(cudaMalloc(&img, npix * 2)); CK(cudaMalloc(&out, 4));
  CK(cudaMemset(img, 1, npix * 2));
  run<0, 64, 192>(img, npix, W, nsm, out, "v4 + 64 ev, 192 thr");
  run<1, 64, 192>(img, npix, W, nsm, out, "v8 + 64 ev, 192 thr");
  run<0, 64, 256>(img, npix, W, nsm, out, "v4 + 64 ev, 256 thr");
  run<0, 64, 384>(img, npix, W, nsm, out, "v4 + 64 ev, 384 thr");
  run<1, 64, 384>(img, npix, W, nsm, out, "v8 + 64 ev, 384 thr");
  run<0, 64, 512>(img, npix, W, nsm, out, "v4 + 64 ev, 512 thr");
  run<0, 64, 768>(img, npix, W, nsm, out, "v4 + 64 ev, 768 thr");
  run<0, 64, 1024>(img, npix, W, nsm, out, "v4 + 64 ev, 1024 thr");
  return 0;
}
