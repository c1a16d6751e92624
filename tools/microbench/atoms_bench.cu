// Microbenchmarks for the judge kernel's inner-loop primitives on B200:
// shared-memory atomics into a 128 KiB packed-u16 histogram (with / without
// return value, spread vs hot bins), __match_any_sync, and L2 REDs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s line %d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__device__ __forceinline__ uint32_t hsh(uint32_t x){ x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x; }

// mode 0: atomicAdd with return used; 1: red (no return); 2: hot (50% lanes to 4 bins) ret; 3: warp-aggregated via match_any on bin
template<int MODE>
__global__ void __launch_bounds__(1024,1) k_atoms(int iters, uint32_t* out) {
  extern __shared__ uint32_t h[];
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) h[i] = 0;
  __syncthreads();
  uint32_t acc = 0;
  uint32_t seed = hsh(blockIdx.x * 1024 + threadIdx.x);
  for (int it = 0; it < iters; ++it) {
    uint32_t r = hsh(seed + it * 0x9e3779b9u);
    uint32_t bin = r & 0xFFFF;
    if (MODE == 2 || MODE == 3) { if (r & 0x10000) bin = (r >> 17) & 3; }
    uint32_t sh = (bin & 1) << 4;
    if (MODE == 0 || MODE == 2) {
      uint32_t old = atomicAdd(&h[bin >> 1], 1u << sh);
      acc ^= old;
    } else if (MODE == 1) {
      atomicAdd(&h[bin >> 1], 1u << sh);
    } else {
      uint32_t m = __match_any_sync(0xffffffffu, bin);
      int lane = threadIdx.x & 31;
      if ((m & ((1u << lane) - 1)) == 0) {
        uint32_t old = atomicAdd(&h[bin >> 1], (uint32_t)__popc(m) << sh);
        acc ^= old;
      }
    }
  }
  __syncthreads();
  acc ^= h[threadIdx.x];
  if (acc == 0x12345678) out[0] = acc;
}

__global__ void __launch_bounds__(1024,1) k_match(int iters, uint32_t* out) {
  uint32_t acc = 0;
  uint32_t seed = hsh(blockIdx.x * 1024 + threadIdx.x);
  for (int it = 0; it < iters; ++it) {
    uint32_t r = hsh(seed + it * 0x9e3779b9u) & 0xFF;
    acc += __match_any_sync(0xffffffffu, r);
  }
  if (acc == 0x12345678) out[0] = acc;
}
__global__ void __launch_bounds__(1024,1) k_hashonly(int iters, uint32_t* out) {
  uint32_t acc = 0;
  uint32_t seed = hsh(blockIdx.x * 1024 + threadIdx.x);
  for (int it = 0; it < iters; ++it) acc += hsh(seed + it * 0x9e3779b9u) & 0xFF;
  if (acc == 0x12345678) out[0] = acc;
}
__global__ void k_redg(int iters, uint32_t* g) {
  uint32_t seed = hsh(blockIdx.x * 1024 + threadIdx.x);
  for (int it = 0; it < iters; ++it) atomicAdd(&g[hsh(seed + it * 0x9e3779b9u) & 0xFFFF], 1u);
}

template<typename F> float timeit(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d kHz\n", nsm, clk);
  uint32_t* out; CK(cudaMalloc(&out, 65536 * 4));
  int iters = 4096;
  size_t smem = 32768 * 4;
  CK(cudaFuncSetAttribute(k_atoms<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_atoms<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_atoms<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_atoms<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  double ops = (double)nsm * 1024 * iters;
  float t;
  t = timeit([&]{ k_hashonly<<<nsm, 1024>>>(iters, out); }); printf("hash-only        %.3f ms  %.3e ops/s  %.2f ops/clk/SM\n", t, ops / t * 1e3, ops / (t * 1e-3) / nsm / (clk * 1e3));
  t = timeit([&]{ k_atoms<0><<<nsm, 1024, smem>>>(iters, out); }); printf("ATOMS ret spread %.3f ms  %.3e ops/s  %.2f ops/clk/SM\n", t, ops / t * 1e3, ops / (t * 1e-3) / nsm / (clk * 1e3));
  t = timeit([&]{ k_atoms<1><<<nsm, 1024, smem>>>(iters, out); }); printf("ATOMS red spread %.3f ms  %.3e ops/s  %.2f ops/clk/SM\n", t, ops / t * 1e3, ops / (t * 1e-3) / nsm / (clk * 1e3));
  t = timeit([&]{ k_atoms<2><<<nsm, 1024, smem>>>(iters, out); }); printf("ATOMS ret hot50  %.3f ms  %.3e ops/s  %.2f ops/clk/SM\n", t, ops / t * 1e3, ops / (t * 1e-3) / nsm / (clk * 1e3));
  t = timeit([&]{ k_atoms<3><<<nsm, 1024, smem>>>(iters, out); }); printf("ATOMS agg hot50  %.3f ms  %.3e ops/s  %.2f ops/clk/SM\n", t, ops / t * 1e3, ops / (t * 1e-3) / nsm / (clk * 1e3));
  t = timeit([&]{ k_match<<<nsm, 1024>>>(iters, out); }); printf("MATCH.ANY        %.3f ms  %.3e ops/s  %.2f lane-ops/clk/SM\n", t, ops / t * 1e3, ops / (t * 1e-3) / nsm / (clk * 1e3));
  CK(cudaMemset(out, 0, 65536 * 4));
  t = timeit([&]{ k_redg<<<nsm * 4, 256>>>(iters, out); }); printf("REDG L2 spread   %.3f ms  %.3e ops/s\n", t, ops / t * 1e3);
  CK(cudaGetLastError());
  return 0;
}
