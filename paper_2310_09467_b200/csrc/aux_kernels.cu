// aux_kernels.cu -- emission, residual image, temporal delta, the composed
// approximate-BWT route, the entropy2d API kernel and the decompression side.
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "entropy.cuh"

namespace pcbz {

// Selected residual stream, row-major, high byte first (core.py:228-237).
__global__ void emit_kernel(const EmitParams P) {
  const int64_t span = P.pix1 - P.pix0;
  const int64_t total = P.nframes * span;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = t / span, k = P.pix0 + (t - f * span);
    const int spec = P.sel[f];
    const uint16_t *src = P.frames + f * P.npix;
    const uint16_t *prv = (spec & 0x80) ? prev_of(P.frames, P.halo, P.npix, f) : nullptr;
    const PredCfg cfg = make_cfg(spec & 0x7F, P.px, P.py);
    const uint32_t r = residual_at(src, prv, P.W, (int)(k / P.W), (int)(k % P.W), cfg);
    P.stream[2 * t] = (uint8_t)(r >> 8);
    P.stream[2 * t + 1] = (uint8_t)r;
  }
}

__global__ void residual_image_kernel(const uint16_t *img, const uint16_t *prev, int64_t h,
                                      int64_t w, int spec, int px, int py, uint16_t *out,
                                      int big_endian) {
  const int64_t total = h * w;
  const PredCfg cfg = make_cfg(spec & 0x7F, px, py);
  const uint16_t *prv = (spec & 0x80) ? prev : nullptr;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t r = residual_at(img, prv, (int)w, (int)(t / w), (int)(t % w), cfg);
    out[t] = big_endian ? (uint16_t)((r >> 8) | ((r & 0xFFu) << 8)) : (uint16_t)r;
  }
}

__global__ void temporal_delta_kernel(const uint16_t *cur, const uint16_t *prev, int64_t n,
                                      uint16_t *out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    out[t] = (uint16_t)(cur[t] - prev[t]);
}

// overlapping byte pairs, first byte high (_kernels.py:116-122)
__global__ void pair_hist_kernel(const uint8_t *s, int64_t n, uint32_t *hist) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t + 1 < n;
       t += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&hist[((uint32_t)s[t] << 8) | s[t + 1]], 1u);
}

// ---- counting_bwt (_kernels.py:93-113) as a stable multi-block counting sort.
// Chunk c of kBwtChunk bytes: counts[v][c] -> exclusive scan in (v, c) order
// gives each chunk's first output slot per byte value; a chunk then scatters
// its predecessors in input order, which keeps the sort stable.
constexpr int kBwtChunk = 2048;

__global__ void bwt_count_kernel(const uint8_t *s, int64_t n, int64_t nchunks, uint32_t *counts) {
  __shared__ uint32_t c[256];
  for (int v = threadIdx.x; v < 256; v += blockDim.x) c[v] = 0;
  __syncthreads();
  const int64_t ch = blockIdx.x;
  const int64_t beg = ch * kBwtChunk, end = min(n, beg + kBwtChunk);
  for (int64_t i = beg + threadIdx.x; i < end; i += blockDim.x) atomicAdd(&c[s[i]], 1u);
  __syncthreads();
  for (int v = threadIdx.x; v < 256; v += blockDim.x) counts[(int64_t)v * nchunks + ch] = c[v];
}

__global__ void bwt_scatter_kernel(const uint8_t *s, int64_t n, int64_t nchunks,
                                   const uint32_t *offsets, uint8_t *out) {
  // one thread per chunk keeps the in-chunk order (not on the timed path)
  const int64_t ch = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (ch >= nchunks) return;
  uint32_t pos[256];
  for (int v = 0; v < 256; ++v) pos[v] = offsets[(int64_t)v * nchunks + ch];
  const int64_t beg = ch * kBwtChunk, end = min(n, beg + kBwtChunk);
  for (int64_t i = beg; i < end; ++i) out[pos[s[i]]++] = s[i == 0 ? n - 1 : i - 1];
}

__global__ void __launch_bounds__(kEntropyThreads) entropy_u64_kernel(const uint64_t *counts, double total,
                                                                    const double *terms, int64_t nterms,
                                                                    double *out) {
  extern __shared__ uint4 smem_raw[];
  NpScratch &scr = *reinterpret_cast<NpScratch *>(smem_raw);
  auto get = [&](int bin) -> uint64_t { return counts[bin]; };
  const double e = block_entropy(get, total, scr, terms, false, nterms);
  if (threadIdx.x == 0) *out = e;
}

__global__ void term_table_kernel(double total, double *terms) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < kTermTable; c += gridDim.x * blockDim.x)
    terms[c] = c == 0 ? 0.0 : np_term((double)c, total);
}

cudaError_t launch_term_table(double total, double *terms, cudaStream_t st) {
  term_table_kernel<<<64, 256, 0, st>>>(total, terms);
  return cudaGetLastError();
}

static int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return (int)g;
}





cudaError_t launch_emit(const EmitParams &p, cudaStream_t st) {
  emit_kernel<<<grid_for(p.nframes * (p.pix1 - p.pix0), 256), 256, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_residual_image(const uint16_t *img, const uint16_t *prev, int64_t h, int64_t w,
                                  int spec, int px, int py, uint16_t *out, int big_endian,
                                  cudaStream_t st) {
  residual_image_kernel<<<grid_for(h * w, 256), 256, 0, st>>>(img, prev, h, w, spec, px, py, out,
                                                              big_endian);
  return cudaGetLastError();
}

cudaError_t launch_temporal_delta(const uint16_t *cur, const uint16_t *prev, int64_t n,
                                  uint16_t *out, cudaStream_t st) {
  temporal_delta_kernel<<<grid_for(n, 256), 256, 0, st>>>(cur, prev, n, out);
  return cudaGetLastError();
}

cudaError_t launch_pair_hist(const uint8_t *s, int64_t n, uint32_t *hist, cudaStream_t st) {
  pair_hist_kernel<<<grid_for(n, 256), 256, 0, st>>>(s, n, hist);
  return cudaGetLastError();
}

size_t counting_bwt_scratch_words(int64_t n) {
  const int64_t nchunks = (n + kBwtChunk - 1) / kBwtChunk;
  size_t temp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, temp, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                (int)(256 * nchunks));
  return (size_t)(2 * 256 * nchunks) + (temp + 3) / 4 + 4;
}

cudaError_t launch_counting_bwt(const uint8_t *s, int64_t n, uint8_t *out, uint32_t *scratch,
                                size_t scratch_words, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t nchunks = (n + kBwtChunk - 1) / kBwtChunk;
  uint32_t *counts = scratch, *offs = scratch + 256 * nchunks;
  void *temp = offs + 256 * nchunks;
  size_t temp_bytes = (scratch_words - 2 * 256 * nchunks) * 4;
  bwt_count_kernel<<<(unsigned)nchunks, 256, 0, st>>>(s, n, nchunks, counts);
  cudaError_t e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, counts, offs,
                                                (int)(256 * nchunks), st);
  if (e != cudaSuccess) return e;
  bwt_scatter_kernel<<<(unsigned)((nchunks + 63) / 64), 64, 0, st>>>(s, n, nchunks, offs, out);
  return cudaGetLastError();
}

cudaError_t launch_entropy_u64(const uint64_t *counts, double total, const double *terms,
                               int64_t nterms, double *out, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    const cudaError_t e = cudaFuncSetAttribute(entropy_u64_kernel,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)sizeof(NpScratch));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  entropy_u64_kernel<<<1, kEntropyThreads, sizeof(NpScratch), st>>>(counts, total, terms, nterms, out);
  return cudaGetLastError();
}



// ---------------------------------------------------------------------------
// decompression side (reference _kernels.py:69-90, predictors.py:101-147)
// ---------------------------------------------------------------------------

// Inverse intra prediction of one frame per CTA.  Every neighbour of (y, x)
// lies on an earlier anti-diagonal (x' + y' < x + y), so the CTA sweeps the
// anti-diagonals in order with a barrier between them.
__global__ void __launch_bounds__(1024) reconstruct_kernel(const uint16_t *res, int64_t h,
                                                           int64_t w, int px, int py,
                                                           const uint8_t *sel, uint16_t *out) {
  const int64_t f = blockIdx.x;
  const int64_t npix = h * w;
  const uint16_t *r = res + f * npix;
  uint16_t *o = out + f * npix;
  const PredCfg c = make_cfg(sel[f] & 0x7F, px, py);
  if (c.grp < 0) {
    for (int64_t i = threadIdx.x; i < npix; i += blockDim.x) o[i] = r[i];
    return;
  }
  const int W = (int)w;
  for (int64_t t = 0; t < h + w - 1; ++t) {
    const int64_t y_lo = t - (w - 1) > 0 ? t - (w - 1) : 0;
    const int64_t y_hi = t < h - 1 ? t : h - 1;
    for (int64_t y = y_lo + threadIdx.x; y <= y_hi; y += blockDim.x) {
      const int x = (int)(t - y);
      int pr = predict_at<false>(o, nullptr, W, (int)y, x, c.sx, c.sy, c.f);
      if (c.grp == 2) pr = (pr + predict_at<false>(o, nullptr, W, (int)y, x, 1, 1, c.f)) >> 1;
      o[y * w + x] = (uint16_t)(r[y * w + x] + pr);
    }
    __syncthreads();
  }
}

// Temporal undelta chain: frame f = inverse_f (+ frame f-1 if temporal).
// Pixels are independent, frames are walked in order by every thread.
__global__ void undelta_chain_kernel(uint16_t *frames, const uint16_t *halo, int64_t nframes,
                                     int64_t npix, const uint8_t *sel) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npix;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t run = halo ? halo[i] : 0u;
    for (int64_t f = 0; f < nframes; ++f) {
      uint32_t v = frames[f * npix + i];
      if (sel[f] & 0x80) v = (v + run) & 0xFFFFu;
      frames[f * npix + i] = (uint16_t)v;
      run = v;
    }
  }
}

cudaError_t launch_reconstruct(const uint16_t *res, const uint16_t *halo, int64_t nframes,
                               int64_t h, int64_t w, int px, int py, const uint8_t *sel,
                               uint16_t *out, cudaStream_t st) {
  reconstruct_kernel<<<(unsigned)nframes, 1024, 0, st>>>(res, h, w, px, py, sel, out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  undelta_chain_kernel<<<grid_for(h * w, 256), 256, 0, st>>>(out, halo, nframes, h * w, sel);
  return cudaGetLastError();
}

}  // namespace pcbz
