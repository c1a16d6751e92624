// common.cuh -- device helpers shared by the judge, emission and decompression
// kernels: neighbour prediction and residuals (reference _kernels.py:31-66).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "judge.cuh"

namespace pcbz {

// Source sample: the frame itself or, for temporal candidates, the modular
// delta against the previous original frame (predictors.py:116-120).
__device__ __forceinline__ int sample_at(const uint16_t *__restrict__ s,
                                         const uint16_t *__restrict__ p, int64_t idx) {
  int v = __ldg(s + idx);
  if (p) v = (v - (int)__ldg(p + idx)) & 0xFFFF;
  return v;
}

// f1..f4 on a neighbour triple; '>> 1' on int32 is floor division for any
// sign, as in the reference (_kernels.py:5-7,31-43).
__device__ __forceinline__ int predict_f(int a, int b, int c, int f) {
  switch (f) {
    case 1: return a + b - c;
    case 2: return a + ((b - c) >> 1);
    case 3: return b + ((a - c) >> 1);
    default: return (a + b) >> 1;
  }
}

// Plain (non read-only-path) loads: used by the decompression sweep, which
// reads pixels written earlier by the same CTA.
template <bool kNc>
__device__ __forceinline__ int load_px(const uint16_t *s, const uint16_t *p, int64_t idx) {
  if constexpr (kNc) return sample_at(s, p, idx);
  else return s[idx];
}

template <bool kNc = true>
__device__ __forceinline__ int predict_at(const uint16_t *s, const uint16_t *p, int W, int y, int x,
                                          int sx, int sy, int f) {
  const int64_t row = (int64_t)y * W;
  const bool left = x >= sx, top = y >= sy;
  const int a = left ? load_px<kNc>(s, p, row + x - sx) : 0;
  const int b = top ? load_px<kNc>(s, p, row - (int64_t)sy * W + x) : 0;
  const int c = (left && top) ? load_px<kNc>(s, p, row - (int64_t)sy * W + x - sx) : 0;
  return predict_f(a, b, c, f);
}

// One residual symbol (_kernels.py:60-65, 179-186).
__device__ __forceinline__ uint32_t residual_at(const uint16_t *s, const uint16_t *p, int W, int y,
                                                int x, const PredCfg &c) {
  const int X = sample_at(s, p, (int64_t)y * W + x);
  if (c.grp < 0) return (uint32_t)X;
  int pr = predict_at(s, p, W, y, x, c.sx, c.sy, c.f);
  if (c.grp == 2) pr = (pr + predict_at(s, p, W, y, x, 1, 1, c.f)) >> 1;
  return (uint32_t)(X - pr) & 0xFFFFu;
}

// (a - b) mod 2^16 in each 16-bit half of a 32-bit word.
__device__ __forceinline__ uint32_t sub16x2(uint32_t a, uint32_t b) {
  return ((a | 0x80008000u) - (b & 0x7FFF7FFFu)) ^ ((a ^ ~b) & 0x80008000u);
}

__device__ __forceinline__ const uint16_t *prev_of(const uint16_t *frames, const uint16_t *halo,
                                                   int64_t npix, int64_t frame) {
  return frame > 0 ? frames + (frame - 1) * npix : halo;
}

}  // namespace pcbz
