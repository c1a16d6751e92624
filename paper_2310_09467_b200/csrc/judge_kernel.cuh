// judge_kernel.cuh -- the sm_100a histogram kernel of the entropy judge
// (instantiated once per fast-path pitch by judge_px.cu).
//
// Semantics follow the reference's fused kernel residual_bwt_pair_hist
// (pkg/src/pcbz/_kernels.py:157-204) and criterion.select_predictor
// (criterion.py:136-173); the parallel decomposition is new:
//
//   * the packed residual stream of one (frame, candidate) pair is cut into
//     segments; one CTA owns a segment, each of its 192 threads owns a
//     contiguous run of pixels and runs the reference's per-key chain
//     automaton (_kernels.py:192-201) on it with a lane-private last-pred
//     table in shared memory -- no cross-lane communication in the hot loop
//     (warp-cooperative matching with __match_any_sync measured 12x slower
//     than a shared atomic on B200, profiles/r01_microbench_atoms_match.log);
//   * fast path (width % 8 == 0, pitch_x <= 16): each lane walks its run in
//     8-pixel chunks with 128-bit read-only loads of the rows it needs and
//     carries left-neighbour history in registers; the pitch is a template
//     parameter, so lenslet-stride neighbours are static register picks;
//   * pair increments go to a CTA-private 65,536-bin histogram of packed u16
//     counters in shared memory (128 KiB); a counter reaching 0x8000 is
//     spilled exactly once (atomicAnd claim) into a small list;
//   * runs are stitched in stream order through their (first, last) pred per
//     key, inside the CTA and then across segments;
//   * the bucket seams of _stitch_buckets (_kernels.py:125-133) close the
//     histogram; entropy.cuh reduces it exactly like the reference's numpy.
#pragma once
#include <utility>

#include "common.cuh"
#include "entropy.cuh"

namespace pcbz {

// ---------------------------------------------------------------------------
// pair -> (frame, candidate)
// ---------------------------------------------------------------------------

struct PairRef {
  int64_t frame;
  int spec;      // predictor byte
  int64_t slot;  // frame * k + index in the full candidate list
};

__device__ __forceinline__ PairRef pair_ref(const JudgeParams &P, int64_t pair) {
  PairRef r;
  if (pair < P.cl.kA) {
    r.frame = 0;
    r.spec = P.cl.byteA[pair];
    r.slot = P.cl.idxA[pair];
  } else {
    const int64_t q = pair - P.cl.kA;
    r.frame = 1 + q / P.cl.kB;
    const int j = (int)(q % P.cl.kB);
    r.spec = P.cl.byteB[j];
    r.slot = r.frame * P.cl.k + P.cl.idxB[j];
  }
  return r;
}

// ---------------------------------------------------------------------------
// chain state of one lane
// ---------------------------------------------------------------------------

struct ChainState {
  uint32_t *hist;   // shared, kHistWords packed u16 counters
  uint32_t hbase;   // shared-window address of hist
  uint32_t lbase;   // shared address of this lane's last-pred column
  uint8_t *F;       // this lane's first-pred row (global scratch)
  uint32_t *spill;  // shared spill list
  int *nspill;
  int *err;
};

// One stream byte as an event (key, pred) of the reference automaton
// (_kernels.py:192-201): pair with the pred of the previous event of the same
// key, or remember pred as the key's first.  The last-pred entry is a u16
// (0x100 = unseen) read and overwritten with independent 16-bit accesses, so
// consecutive events do not wait on each other's shared-memory latency.
// Returns the incremented bin (or ~0u) and ORs the counter's toggled bits
// into `flag`: bit 15 of a half toggles exactly when that counter crosses
// 0x7FFF -> 0x8000.
__device__ __forceinline__ uint32_t chain_event(const ChainState &cs, uint32_t key, uint32_t pred,
                                                uint32_t &flag) {
  const uint32_t a = cs.lbase + (key >> 1) * (4u * kJudgeThreads) + ((key & 1u) << 1);
  uint32_t last;
  asm volatile("ld.shared.u16 %0, [%1];" : "=r"(last) : "r"(a));
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "r"(pred));
  if (last == kUnseen) {
    cs.F[key] = (uint8_t)pred;
    return ~0u;
  }
  const uint32_t bin = (last << 8) | pred;
  const uint32_t inc = 1u << ((pred & 1u) << 4);
  const uint32_t old = atomicAdd(&cs.hist[bin >> 1], inc);
  flag |= old ^ (old + inc);
  return bin;
}

// Move 0x8000 out of `bin`'s counter if its bit 15 is set.  atomicAnd makes
// exactly one claimant per crossing; counts are never lost or doubled.
__device__ __forceinline__ void claim_spill(const ChainState &cs, uint32_t bin) {
  if (bin == ~0u) return;
  const uint32_t m = 0x8000u << ((bin & 1u) << 4);
  const uint32_t old = atomicAnd(&cs.hist[bin >> 1], ~m);
  if (old & m) {
    const int i = atomicAdd(cs.nspill, 1);
    if (i < kSpillCap) cs.spill[i] = bin;
    else atomicExch(cs.err, 2);
  }
}

// increment outside the hot loop (stitching): claim immediately
__device__ __forceinline__ void hist_inc_now(const ChainState &cs, uint32_t bin) {
  const uint32_t inc = 1u << ((bin & 1u) << 4);
  const uint32_t old = atomicAdd(&cs.hist[bin >> 1], inc);
  if ((old ^ (old + inc)) & 0x80008000u) claim_spill(cs, bin);
}

// ---------------------------------------------------------------------------
// generic lane: any width / pitch, one pixel at a time
// ---------------------------------------------------------------------------

static __device__ void lane_generic(const uint16_t *src, const uint16_t *prv, const PredCfg &cfg, int W,
                             int64_t npix, int64_t a, int64_t b, const ChainState &cs) {
  if (a >= b) return;
  const int64_t q = a > 0 ? a - 1 : npix - 1;  // wrap predecessor (_kernels.py:172-190)
  uint32_t prev_lo = residual_at(src, prv, W, (int)(q / W), (int)(q % W), cfg) & 0xFFu;
  int y = (int)(a / W), x = (int)(a % W);
  uint32_t flag = 0;
  for (int64_t k = a; k < b; ++k) {
    const uint32_t r = residual_at(src, prv, W, y, x, cfg);
    const uint32_t hi = r >> 8, lo = r & 0xFFu;
    const uint32_t b0 = chain_event(cs, hi, prev_lo, flag);
    const uint32_t b1 = chain_event(cs, lo, hi, flag);
    if (flag & 0x80008000u) {
      claim_spill(cs, b0);
      claim_spill(cs, b1);
    }
    flag = 0;
    prev_lo = lo;
    if (++x == W) { x = 0; ++y; }
  }
}

// ---------------------------------------------------------------------------
// fast lane: 8-pixel chunks, 128-bit loads, register neighbour history
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint4 ld_chunk(const uint16_t *__restrict__ s,
                                          const uint16_t *__restrict__ p, int64_t off) {
  uint4 a = __ldg(reinterpret_cast<const uint4 *>(s + off));
  if (p) {
    const uint4 b = __ldg(reinterpret_cast<const uint4 *>(p + off));
    a.x = sub16x2(a.x, b.x); a.y = sub16x2(a.y, b.y);
    a.z = sub16x2(a.z, b.z); a.w = sub16x2(a.w, b.w);
  }
  return a;
}

__device__ __forceinline__ void unpack8(const uint4 &w, int (&v)[8]) {
  v[0] = w.x & 0xFFFF; v[1] = w.x >> 16; v[2] = w.y & 0xFFFF; v[3] = w.y >> 16;
  v[4] = w.z & 0xFFFF; v[5] = w.z >> 16; v[6] = w.w & 0xFFFF; v[7] = w.w >> 16;
}

// f1..f4 of the reference (_kernels.py:36-43), compile-time function id
template <int F>
__device__ __forceinline__ int pred_f(int A, int B, int C) {
  if constexpr (F == 1) return A + B - C;
  else if constexpr (F == 2) return A + ((B - C) >> 1);
  else if constexpr (F == 3) return B + ((A - C) >> 1);
  else return (A + B) >> 1;
}

__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

__device__ __forceinline__ void sts_u16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "r"(v));
}

// explicit shared-window atomics: the lane functions are not inlined into the
// kernel, so generic pointers would compile to (slow) generic ATOM
__device__ __forceinline__ uint32_t atoms_add(uint32_t a, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v));
  return old;
}

__device__ __forceinline__ uint32_t atoms_and(uint32_t a, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.and.b32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v));
  return old;
}

// Clear bits 15/31 of a histogram word and spill 0x8000 for each that was
// set.  Any claimant may clear any set bit: atomicAnd makes every clear
// unique, so counts are transferred exactly once.
__device__ __forceinline__ void claim_word(const ChainState &cs, uint32_t word) {
  const uint32_t old = atoms_and(cs.hbase + 4u * word, ~0x80008000u);
  if (old & 0x80008000u) {
    const int n = (old & 0x8000u ? 1 : 0) + (old & 0x80000000u ? 1 : 0);
    const int i = atomicAdd(cs.nspill, n);
    if (i + n <= kSpillCap) {
      int j = i;
      if (old & 0x8000u) cs.spill[j++] = 2 * word;
      if (old & 0x80000000u) cs.spill[j] = 2 * word + 1;
    } else {
      atomicExch(cs.err, 2);
    }
  }
}

// One lane's run of `nch` 8-pixel chunks starting at pixel a (a % 8 == 0),
// for intra predictor ID and lenslet pitch PX (both compile-time).
//
// Per chunk the 16 stream bytes become 16 events (key, pred):
//   e = 2i: (hi_i, lo_{i-1})     e = 2i + 1: (lo_i, hi_i)      (_kernels.py:187-202)
// Phase A performs the 16 last-pred lookups/updates in stream order (each an
// independent 16-bit load + store, no read-modify-write); phase B issues
// the 16 histogram atomics.  A counter whose bit 15 is found set in an
// atomic's returned word is claimed at the end of the chunk; the kernel
// sweeps the histogram once more after the loop for any crossing nobody
// observed.  First occurrences (pred -> first-pred row) are rare after a
// run's warm-up and handled off the common path.
template <int PX, int ID>
__device__ __noinline__ void lane_fast(const uint16_t *__restrict__ src,
                                       const uint16_t *__restrict__ prv, int W, int py,
                                       int64_t npix, int64_t a, int64_t nch, const PredCfg cfg,
                                       const ChainState cs) {
  constexpr int GRP = ID == 0 ? -1 : (ID - 1) / 4;
  constexpr int F = ID == 0 ? 0 : (ID - 1) % 4 + 1;
  constexpr bool kT1 = GRP == 0 || GRP == 2;  // row y-1   (pixel-adjacent B, C)
  constexpr bool kTS = GRP == 1 || GRP == 2;  // row y-py  (lenslet B, C)
  constexpr bool kXH = GRP >= 0;              // left history of row y
  constexpr bool kXH2 = kTS && PX > 8;        // second chunk of history
  if (nch <= 0) return;
  const int64_t q = a > 0 ? a - 1 : npix - 1;  // wrap predecessor (_kernels.py:172-190)
  uint32_t prev_lo = residual_at(src, prv, W, (int)(q / W), (int)(q % W), cfg) & 0xFFu;
  int y = (int)(a / W), x0 = (int)(a % W);
  const uint4 Z = make_uint4(0, 0, 0, 0);
  auto row = [&](int yy) -> int64_t { return (int64_t)yy * W; };
  uint4 Xh1 = Z, Xh2 = Z, T1h = Z, TSh1 = Z, TSh2 = Z;
  if (x0 > 0) {  // history of a run that starts mid-row
    if (kXH) Xh1 = ld_chunk(src, prv, row(y) + x0 - 8);
    if (kXH2 && x0 >= 16) Xh2 = ld_chunk(src, prv, row(y) + x0 - 16);
    if (kT1 && y >= 1) T1h = ld_chunk(src, prv, row(y - 1) + x0 - 8);
    if (kTS && y >= py) {
      TSh1 = ld_chunk(src, prv, row(y - py) + x0 - 8);
      if (kXH2 && x0 >= 16) TSh2 = ld_chunk(src, prv, row(y - py) + x0 - 16);
    }
  }
  uint4 cX = ld_chunk(src, prv, row(y) + x0);
  uint4 cT1 = (kT1 && y >= 1) ? ld_chunk(src, prv, row(y - 1) + x0) : Z;
  uint4 cTS = (kTS && y >= py) ? ld_chunk(src, prv, row(y - py) + x0) : Z;
  for (int64_t c = 0; c < nch; ++c) {
    int ny = y, nx = x0 + 8;
    if (nx == W) { nx = 0; ++ny; }
    uint4 nX = Z, nT1 = Z, nTS = Z;
    if (c + 1 < nch) {  // prefetch the next chunk
      nX = ld_chunk(src, prv, row(ny) + nx);
      if (kT1 && ny >= 1) nT1 = ld_chunk(src, prv, row(ny - 1) + nx);
      if (kTS && ny >= py) nTS = ld_chunk(src, prv, row(ny - py) + nx);
    }
    // ---- residuals of the 8 pixels (_kernels.py:179-186) --------------------
    uint32_t r[8];
    {
      int X[8], T1[8], TS[8], H1[8], H2[8], S1[8], S2[8], t1h[8];
      unpack8(cX, X);
      if (kT1) { unpack8(cT1, T1); unpack8(T1h, t1h); }
      if (kTS) { unpack8(cTS, TS); unpack8(TSh1, S1); }
      if (kXH) unpack8(Xh1, H1);
      if (kXH2) { unpack8(Xh2, H2); unpack8(TSh2, S2); }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if constexpr (GRP < 0) {
          r[i] = (uint32_t)X[i];
        } else {
          int p = 0, p1 = 0;
          if constexpr (kT1) {  // pixel-adjacent neighbours (1, 1)
            p1 = pred_f<F>(i ? X[i - 1] : H1[7], T1[i], i ? T1[i - 1] : t1h[7]);
          }
          if constexpr (kTS) {  // lenslet-stride neighbours (PX, py)
            const int qq = i - PX;
            int A, C;
            if (qq >= 0) { A = X[qq]; C = TS[qq]; }
            else if (qq >= -8) { A = H1[qq + 8]; C = S1[qq + 8]; }
            else { A = H2[qq + 16]; C = S2[qq + 16]; }
            const int p2 = pred_f<F>(A, TS[i], C);
            p = GRP == 2 ? ((p1 + p2) >> 1) : p2;  // phase group (_kernels.py:63-64)
          } else {
            p = p1;
          }
          r[i] = (uint32_t)(X[i] - p) & 0xFFFFu;
        }
      }
    }
    // ---- events ---------------------------------------------------------------
    uint32_t key[16], prd[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      key[2 * i] = r[i] >> 8;
      prd[2 * i] = i ? (r[i - 1] & 0xFFu) : prev_lo;
      key[2 * i + 1] = r[i] & 0xFFu;
      prd[2 * i + 1] = r[i] >> 8;
    }
    prev_lo = r[7] & 0xFFu;
    uint32_t last[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {  // phase A: in stream order
      const uint32_t la = cs.lbase + key[e] * 2u + (key[e] >> 1) * (4u * kJudgeThreads - 4u);
      last[e] = lds_u16(la);
      sts_u16(la, prd[e]);
    }
    // phase B: one unconditional atomic per event.  A first occurrence has
    // last == 0x100, i.e. bin 0x100xx: it lands in the dummy row past the
    // histogram and is excluded from every count.
    uint32_t flag = 0, fresh = 0, word[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      fresh |= last[e];
      word[e] = last[e] * 128u + (prd[e] >> 1);  // bin = last * 256 + pred, 2 bins/word
      flag |= atoms_add(cs.hbase + 4u * word[e], 1u + (prd[e] & 1u) * 0xFFFFu);
    }
    if (fresh & kUnseen) {  // first occurrence of a key in this run
#pragma unroll
      for (int e = 0; e < 16; ++e)
        if (last[e] == kUnseen) cs.F[key[e]] = (uint8_t)prd[e];
    }
    if (flag & 0x80008000u) {  // some counter has crossed 0x8000: claim
#pragma unroll
      for (int e = 0; e < 16; ++e)
        if (word[e] < (uint32_t)kHistWords) claim_word(cs, word[e]);
    }
    if (nx == 0) {
      Xh1 = Xh2 = T1h = TSh1 = TSh2 = Z;  // new row: left neighbours are 0
    } else {
      Xh2 = Xh1; Xh1 = cX; T1h = cT1; TSh2 = TSh1; TSh1 = cTS;
    }
    y = ny; x0 = nx;
    cX = nX; cT1 = nT1; cTS = nTS;
  }
}

template <int PX, int... IDs>
__device__ __forceinline__ void lane_fast_dispatch(int id, const uint16_t *src,
                                                   const uint16_t *prv, int W, int py,
                                                   int64_t npix, int64_t a, int64_t nch,
                                                   const PredCfg &cfg, const ChainState &cs,
                                                   std::integer_sequence<int, IDs...>) {
  ((id == IDs ? lane_fast<PX, IDs>(src, prv, W, py, npix, a, nch, cfg, cs) : void()), ...);
}

// ---------------------------------------------------------------------------
// the judge kernel: persistent CTAs pull (pair, segment) items
// ---------------------------------------------------------------------------
//
// dynamic shared memory:
//   hist   kHistWords            packed u16 counters
//   last   kLastWords * 192      last-pred tables, word (key>>1)*192 + lane
//   spill  kSpillCap             spilled bins
// after the hot loop the last-pred region is reused for the spilled-bin
// bitmap (words [0, 2048)), first/last per key ([2048, 2560)) and the
// entropy scratch ([2560, ...)).

template <int PX>
__global__ void __launch_bounds__(kJudgeThreads, 1) judge_hist_kernel(const JudgeParams P) {
  extern __shared__ uint4 smem_raw[];
  uint32_t *hist_w = reinterpret_cast<uint32_t *>(smem_raw);
  uint32_t *last_w = hist_w + kHistWords + kDummyWords;
  uint32_t *spill_w = last_w + kLastWords * kJudgeThreads;
  __shared__ int s_item, s_nspill;
  int *s_first = reinterpret_cast<int *>(last_w) + 2048;
  int *s_last = s_first + 256;
  NpScratch &scr = *reinterpret_cast<NpScratch *>(last_w + 2560);

  const int tid = threadIdx.x;
  const int64_t nitems = P.npairs * P.S;
  ChainState cs;
  cs.hist = hist_w;
  cs.hbase = (uint32_t)__cvta_generic_to_shared(hist_w);
  cs.lbase = (uint32_t)__cvta_generic_to_shared(last_w + tid);
  cs.F = P.fscratch + ((size_t)blockIdx.x * kJudgeThreads + tid) * 256;
  cs.spill = spill_w;
  cs.nspill = &s_nspill;
  cs.err = P.err;
  const uint8_t *Fcta = P.fscratch + (size_t)blockIdx.x * kJudgeThreads * 256;
  uint32_t *Llane = last_w + tid;

  for (;;) {
    if (tid == 0) {
      s_item = atomicAdd(P.counter, 1);
      s_nspill = 0;
    }
    uint4 *h4 = reinterpret_cast<uint4 *>(hist_w);
    for (int i = tid; i < (kHistWords + kDummyWords) / 4; i += kJudgeThreads) h4[i] = make_uint4(0, 0, 0, 0);
    for (int w = 0; w < kLastWords; ++w) Llane[w * kJudgeThreads] = kUnseen | (kUnseen << 16);
    __syncthreads();
    const int64_t item = s_item;
    if (item >= nitems) break;

    const int64_t pair = item / P.S;
    const int seg = (int)(item % P.S);
    const PairRef pr = pair_ref(P, pair);
    const uint16_t *src = P.frames + pr.frame * P.npix;
    const uint16_t *prv = (pr.spec & 0x80) ? prev_of(P.frames, P.halo, P.npix, pr.frame) : nullptr;
    const PredCfg cfg = make_cfg(pr.spec & 0x7F, P.px, P.py);

    if constexpr (PX > 0) {
      // chunk-granular segments and runs
      const int64_t nchunk = P.npix / 8;
      const int64_t cb = nchunk * seg / P.S, ce = nchunk * (seg + 1) / P.S;
      const int64_t ca = cb + (ce - cb) * tid / kJudgeThreads;
      const int64_t cz = cb + (ce - cb) * (tid + 1) / kJudgeThreads;
      lane_fast_dispatch<PX>(pr.spec & 0x7F, src, prv, P.W, P.py, P.npix, ca * 8, cz - ca, cfg, cs,
                             std::make_integer_sequence<int, 13>{});
    } else {
      const int64_t sb = P.npix * seg / P.S, se = P.npix * (seg + 1) / P.S;
      const int64_t len = se - sb;
      lane_generic(src, prv, cfg, P.W, P.npix, sb + len * tid / kJudgeThreads,
                   sb + len * (tid + 1) / kJudgeThreads, cs);
    }
    __syncthreads();
    for (int w = tid; w < kHistWords; w += kJudgeThreads)
      if (hist_w[w] & 0x80008000u) claim_word(cs, (uint32_t)w);
    __syncthreads();

    // ---- stitch the 192 runs in stream order (segment-summary combine) -----
    int my_first0 = -1, my_last0 = -1, my_first1 = -1, my_last1 = -1;
    for (int v = tid, i = 0; v < 256; v += kJudgeThreads, ++i) {
      int carried = -1, first = -1;
      const uint32_t *col = last_w + (v >> 1) * kJudgeThreads;
      const uint32_t sh = (v & 1) << 4;
      for (int j = 0; j < kJudgeThreads; ++j) {
        const uint32_t e = (col[j] >> sh) & 0xFFFFu;
        const uint32_t f = Fcta[(size_t)j * 256 + v];
        if (e != kUnseen) {
          if (carried >= 0) hist_inc_now(cs, ((uint32_t)carried << 8) | f);
          else first = (int)f;
          carried = (int)e;
        }
      }
      if (i == 0) { my_first0 = first; my_last0 = carried; }
      else { my_first1 = first; my_last1 = carried; }
    }
    __syncthreads();
    s_first[tid] = my_first0;
    s_last[tid] = my_last0;
    if (tid + kJudgeThreads < 256) {
      s_first[tid + kJudgeThreads] = my_first1;
      s_last[tid + kJudgeThreads] = my_last1;
    }
    __syncthreads();

    if (P.direct) {
      // whole stream in this CTA: bucket seams (_kernels.py:125-133) ...
      if (tid == 0) {
        int carried = -1;
        for (int v = 0; v < 256; ++v) {
          if (s_first[v] < 0) continue;
          if (carried >= 0) hist_inc_now(cs, ((uint32_t)carried << 8) | (uint32_t)s_first[v]);
          carried = s_last[v];
        }
      }
      __syncthreads();
      // ... spilled bins marked in a bitmap, then the entropy
      uint32_t *spilled = last_w;
      for (int i = tid; i < 2048; i += kJudgeThreads) spilled[i] = 0;
      __syncthreads();
      const int ns = min(s_nspill, kSpillCap);
      for (int i = tid; i < ns; i += kJudgeThreads)
        atomicOr(&spilled[spill_w[i] >> 5], 1u << (spill_w[i] & 31));
      __syncthreads();
      auto get = [&](int bin) -> double {
        uint32_t c = (hist_w[bin >> 1] >> ((bin & 1) << 4)) & 0xFFFFu;
        if (spilled[bin >> 5] & (1u << (bin & 31)))
          for (int i = 0; i < ns; ++i) c += spill_w[i] == (uint32_t)bin ? kSpill : 0u;
        return (double)c;
      };
      const double e = block_entropy(get, (double)(2 * P.npix - 1), scr);
      if (tid == 0) P.ent[pr.slot] = e;
    } else {
      // flush into the pair's global histogram and publish the summary
      uint32_t *G = P.ghist + (size_t)pr.slot * 65536;
      for (int w = tid; w < kHistWords; w += kJudgeThreads) {
        const uint32_t v = hist_w[w];
        if (v & 0xFFFFu) atomicAdd(&G[2 * w], v & 0xFFFFu);
        if (v >> 16) atomicAdd(&G[2 * w + 1], v >> 16);
      }
      const int ns = min(s_nspill, kSpillCap);
      for (int i = tid; i < ns; i += kJudgeThreads) atomicAdd(&G[spill_w[i]], kSpill);
      int16_t *sum = P.segsum + ((size_t)pr.slot * P.S + seg) * 512;
      for (int v = tid; v < 256; v += kJudgeThreads) {
        sum[v] = (int16_t)s_first[v];
        sum[256 + v] = (int16_t)s_last[v];
      }
    }
    __syncthreads();
  }
}


}  // namespace pcbz
