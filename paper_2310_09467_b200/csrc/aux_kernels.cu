// aux_kernels.cu -- emission, residual image, temporal delta, the composed
// approximate-BWT route, the entropy2d API kernel and the decompression side.
#include <algorithm>
#include <utility>
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

// (F - P) mod 2^16 of pixels [pix0, pix1) of frames f0.. (8-aligned), 8 pixels
// per thread (predictors.py:116-120)
__global__ void delta_frames_kernel(const uint16_t *frames, const uint16_t *halo, int64_t nframes,
                                    int64_t npix, int64_t f0, int64_t pix0, int64_t pix1, uint16_t *delta) {
  const int64_t per = (pix1 - pix0) / 8;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (nframes - f0) * per;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = f0 + t / per, i = pix0 + (t % per) * 8;
    const uint16_t *cur = frames + f * npix, *prv = f > 0 ? frames + (f - 1) * npix : halo;
    const uint4 a = __ldg(reinterpret_cast<const uint4 *>(cur + i));
    const uint4 b = __ldg(reinterpret_cast<const uint4 *>(prv + i));
    *reinterpret_cast<uint4 *>(delta + f * npix + i) =
        make_uint4(sub16x2(a.x, b.x), sub16x2(a.y, b.y), sub16x2(a.z, b.z), sub16x2(a.w, b.w));
  }
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

cudaError_t launch_delta_frames(const uint16_t *frames, const uint16_t *halo, int64_t nframes,
                                int64_t npix, int64_t f0, int64_t pix0, int64_t pix1, uint16_t *delta,
                                cudaStream_t st) {
  if (nframes <= f0 || pix1 <= pix0) return cudaSuccess;
  delta_frames_kernel<<<grid_for((nframes - f0) * ((pix1 - pix0) / 8), 256), 256, 0, st>>>(
      frames, halo, nframes, npix, f0, pix0, pix1, delta);
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

// Inverse intra prediction as a pipelined wavefront over 32-row bands (one
// warp per band, lane = row): lane r handles column s - r at step s, so the
// neighbours up (row r - sy, same column) and left (own row, column - sx)
// were computed at an earlier step of the same warp and sit in a per-warp
// shared-memory ring of the band's rows; rows above the band come from the
// band above, copied into the ring's halo rows once per 32 steps after its
// published progress covers them.  Units (frame, band) are grabbed
// band-major, so a band only ever waits on a band grabbed before it (no
// deadlock); a band runs ~64 steps behind the band above, so a 2048^2 frame
// is ~6,200 dependent steps deep instead of 4,095 CTA-wide barriers.
// Pitches px <= 64, py <= 31 (the ring holds 128 columns, the halo 32 rows).
constexpr int kRecWarps = 4;
constexpr int kRecRing = 128;
constexpr int kRecRows = 64;   // 32 halo rows + the band's 32 rows
constexpr size_t kRecSmemBytes = (size_t)kRecWarps * kRecRows * kRecRing * sizeof(uint16_t);

__device__ __forceinline__ int64_t mn64(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ int64_t mx64(int64_t a, int64_t b) { return a > b ? a : b; }

__device__ __forceinline__ int ld_acquire_i32(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_i32(int *p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// One band (32 rows from row 32 * b) of one frame; GRP / F compile-time
// (make_cfg), columns in 32-bit.
template <int GRP, int F>
__device__ __forceinline__ void reconstruct_band(const uint16_t *__restrict__ R, uint16_t *O, int h, int w,
                                                 int px, int py, int b, int *pg,
                                                 uint16_t (*rg)[kRecRing], int lane) {
  constexpr int kMask = kRecRing - 1;
  const int sx = GRP == 0 ? 1 : px, sy = GRP == 0 ? 1 : py;
  const int dy_max = GRP == 2 ? max(py, 1) : sy;
  const int y = b * 32 + lane;
  const bool row_ok = y < h;
  const uint16_t *Rrow = R + (int64_t)(row_ok ? y : 0) * w;
  const uint16_t *own = rg[32 + lane];
  const uint16_t *up = rg[32 + lane - sy];
  const uint16_t *up1 = rg[32 + lane - 1];
  const bool top = y >= sy, top1 = y >= 1;
  for (int s0 = 0; s0 < w + 31; s0 += 32) {
    if (b > 0) {
      // rows above: the band above must have finished columns < s0 + 33
      const int need = min(w, s0 + 33);
      if (lane == 0)
        while (ld_acquire_i32(pg + b - 1) < need) __nanosleep(32);
      __syncwarp();
      // only this block's 32 new columns: earlier ones are in the ring
      // already (final when copied), and the ring keeps 128 columns
      const int x = s0 + lane;
      if (x < w) {
        uint16_t v[31];
#pragma unroll
        for (int i = 0; i < 31; ++i)
          v[i] = i < dy_max ? __ldcg(O + (int64_t)(b * 32 - dy_max + i) * w + x) : 0;
#pragma unroll
        for (int i = 0; i < 31; ++i)
          if (i < dy_max) rg[32 - dy_max + i][x & kMask] = v[i];
      }
      __syncwarp();
    }
    uint32_t rr[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int x = s0 + j - lane;
      rr[j] = (row_ok && x >= 0 && x < w) ? __ldg(Rrow + x) : 0u;
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int x = s0 + j - lane;
      if (row_ok && x >= 0 && x < w) {
        const bool left = x >= sx;
        const int A = left ? own[(x - sx) & kMask] : 0;
        const int B = top ? up[x & kMask] : 0;
        const int C = (left && top) ? up[(x - sx) & kMask] : 0;
        int pr;
        if constexpr (F == 1) pr = A + B - C;
        else if constexpr (F == 2) pr = A + ((B - C) >> 1);
        else if constexpr (F == 3) pr = B + ((A - C) >> 1);
        else pr = (A + B) >> 1;
        if constexpr (GRP == 2) {  // phase: average with the pixel-adjacent prediction
          const bool l1 = x >= 1;
          const int a1 = l1 ? own[(x - 1) & kMask] : 0;
          const int b1 = top1 ? up1[x & kMask] : 0;
          const int c1 = (l1 && top1) ? up1[(x - 1) & kMask] : 0;
          int p1;
          if constexpr (F == 1) p1 = a1 + b1 - c1;
          else if constexpr (F == 2) p1 = a1 + ((b1 - c1) >> 1);
          else if constexpr (F == 3) p1 = b1 + ((a1 - c1) >> 1);
          else p1 = (a1 + b1) >> 1;
          pr = (pr + p1) >> 1;
        }
        rg[32 + lane][x & kMask] = (uint16_t)(rr[j] + (uint32_t)pr);
      }
      __syncwarp();
    }
    // the block's 32 new columns of every row, stored row by row with the
    // lanes along the columns (coalesced), then published
    for (int i = 0; i < 32; ++i) {
      const int x = s0 - i + lane;
      if (b * 32 + i < h && x >= 0 && x < w) O[(int64_t)(b * 32 + i) * w + x] = rg[32 + i][x & kMask];
    }
    __syncwarp();
    // row 31 has finished columns < s0 + 1; rows above it are further on
    if (lane == 31) {
      __threadfence();
      st_release_i32(pg + b, min(w, max(0, s0 + 1)));
    }
  }
}

template <int... IDs>
__device__ __forceinline__ void reconstruct_band_dispatch(int id, const uint16_t *R, uint16_t *O, int h, int w,
                                                          int px, int py, int b, int *pg,
                                                          uint16_t (*rg)[kRecRing], int lane,
                                                          std::integer_sequence<int, IDs...>) {
  ((id == IDs ? reconstruct_band<(IDs - 1) / 4, (IDs - 1) % 4 + 1>(R, O, h, w, px, py, b, pg, rg, lane)
              : void()), ...);
}

__global__ void __launch_bounds__(32 * kRecWarps, 3) reconstruct_bands_kernel(
    const uint16_t *res, int h, int w, int px, int py, const uint8_t *sel, uint16_t *out,
    int64_t nframes, int nbands, int *prog, unsigned long long *counter) {
  extern __shared__ uint16_t rec_smem[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint16_t(*rg)[kRecRing] = reinterpret_cast<uint16_t(*)[kRecRing]>(rec_smem + (size_t)wid * kRecRows * kRecRing);
  const int64_t npix = (int64_t)h * w;
  const int64_t units = nframes * nbands;
  for (;;) {
    unsigned long long u = 0;
    if (lane == 0) u = atomicAdd(counter, 1ull);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u >= (unsigned long long)units) break;
    const int b = (int)(u / nframes);
    const int64_t f = (int64_t)(u % nframes);
    const int id = sel[f] & 0x7F;
    const uint16_t *R = res + f * npix;
    uint16_t *O = out + f * npix;
    int *pg = prog + f * nbands;
    if (id == 0) {  // identity: no dependencies; the band's rows, 16 bytes per lane
      const int64_t r0 = (int64_t)b * 32 * w, r1 = min((int64_t)(b + 1) * 32 * w, npix);
      if ((((uintptr_t)R | (uintptr_t)O) & 15) == 0 && (r0 & 7) == 0) {
        const int64_t v1 = r0 + ((r1 - r0) & ~(int64_t)7);
        for (int64_t i = r0 + 8 * lane; i < v1; i += 256)
          *reinterpret_cast<uint4 *>(O + i) = __ldg(reinterpret_cast<const uint4 *>(R + i));
        for (int64_t i = v1 + lane; i < r1; i += 32) O[i] = R[i];
      } else {
        for (int64_t i = r0 + lane; i < r1; i += 32) O[i] = R[i];
      }
    } else {
      reconstruct_band_dispatch(id, R, O, h, w, px, py, b, pg, rg, lane,
                                std::integer_sequence<int, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12>{});
    }
    __syncwarp();
    if (lane == 31) {
      __threadfence();
      st_release_i32(pg + b, w);
    }
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
  cudaError_t e;
  const int64_t nbands = (h + 31) / 32;
  if (px <= 64 && py <= 31 && w < (1ll << 30) && h < (1ll << 30) && nframes * nbands < (1ll << 40)) {
    static bool configured = false;
    if (!configured) {
      e = cudaFuncSetAttribute(reconstruct_bands_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)kRecSmemBytes);
      if (e != cudaSuccess) return e;
      configured = true;
    }
    // progress words (one per band) + the unit counter, stream-ordered scratch
    const size_t words = (size_t)nframes * nbands;
    char *scratch = nullptr;
    if ((e = cudaMallocAsync(reinterpret_cast<void **>(&scratch), words * 4 + 16, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(scratch, 0, words * 4 + 16, st)) != cudaSuccess) return e;
    int *prog = reinterpret_cast<int *>(scratch + 16);
    auto *counter = reinterpret_cast<unsigned long long *>(scratch);
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    // persistent grid (3 CTAs of 64 KiB per SM); units are grabbed by running
    // warps only, so a waiting band's predecessor is always being worked on
    const int64_t want = (words + kRecWarps - 1) / kRecWarps;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)nsm * 3));
    reconstruct_bands_kernel<<<grid, 32 * kRecWarps, kRecSmemBytes, st>>>(res, (int)h, (int)w, px, py, sel, out,
                                                                         nframes, (int)nbands, prog, counter);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = cudaFreeAsync(scratch, st)) != cudaSuccess) return e;
  } else {
    reconstruct_kernel<<<(unsigned)nframes, 1024, 0, st>>>(res, h, w, px, py, sel, out);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  undelta_chain_kernel<<<grid_for(h * w, 256), 256, 0, st>>>(out, halo, nframes, h * w, sel);
  return cudaGetLastError();
}

}  // namespace pcbz
