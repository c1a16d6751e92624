// entropy.cuh -- block-wide fp64 entropy that reproduces the reference's
// numpy evaluation bit for bit (criterion.py:86-96):
//
//     counts = hist.counts[hist.counts > 0]      # occupied bins, bin order
//     p = counts / float(hist.total)
//     E = float(-(p * np.log2(p)).sum())
//
// np.sum over a contiguous float64 array is numpy's pairwise summation:
// n < 8 -> sequential from -0.0; n <= 128 -> eight interleaved accumulators
// combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) then the n % 8 tail;
// otherwise split at n/2 rounded down to a multiple of 8 and recurse (numpy
// _core/src/umath/loops_utils.h.src; the leaf/fold decomposition below is
// checked bit-for-bit against np.sum for n = 1..65536 in
// tests/test_entropy_emulation.py).  Every term is rounded exactly like
// numpy's (IEEE division, device log2, IEEE product -- explicit _rn
// intrinsics so nvcc cannot contract them into FMAs), so the device entropy
// equals the reference's whenever log2 rounds alike (both are correctly
// rounded for nearly all arguments), and mathematically tied candidates tie
// or break exactly as in the reference.
//
// Parallel form: an occupancy bitmap (warp ballots); thread t owns a run of
// 32-bin occupancy words; a block scan of occupied counts gives every occupied bin its index in the
// (virtual) compacted term array.  The recursion tree is built breadth-first
// by one warp (ballot compaction per level); all leaves (index ranges of at
// most 128 terms) are evaluated in parallel by walking the occupancy bitmap;
// internal nodes are then folded bottom-up one level at a time.  Each
// internal node's value is left + right exactly as in the recursion, so the
// evaluation order across nodes does not matter.
#pragma once
#include <cstdint>

#include "judge.cuh"

namespace pcbz {

constexpr int kNpBlock = 128;      // numpy PW_BLOCKSIZE
constexpr int kOccWords = 2048;    // 65536 bins / 32
constexpr int kNpNodeMax = 2048;   // <= 1024 leaves (>= 64 terms each once n > 128) + internals
constexpr int kNpLevelMax = 16;
constexpr uint32_t kNpLeaf = 0xFFFFFFFFu;

// scratch of a block of NT threads
template <int NT>
struct NpScratchT {
  uint32_t off[NT + 1];               // compacted index of each thread's first term
  uint32_t occ[kOccWords];            // occupancy bitmap
  uint32_t node_beg[kNpNodeMax];
  uint32_t node_len[kNpNodeMax];
  uint32_t node_child[kNpNodeMax];    // index of the left child (right = +1), or kNpLeaf
  double node_sum[kNpNodeMax];
  uint32_t level_start[kNpLevelMax + 1];
  int nlevels;
};
using NpScratch = NpScratchT<kEntropyThreads>;

// first occupancy word of thread t's run (a block of NT threads)
template <int NT>
__device__ __forceinline__ int occ_word_lo(int t) { return (kOccWords * t) / NT; }

// Breadth-first recursion tree of numpy's pairwise sum over n terms; one warp.
template <typename Scratch>
__device__ inline void np_build_tree(uint32_t n, Scratch &S) {
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    S.node_beg[0] = 0;
    S.node_len[0] = n;
    S.level_start[0] = 0;
    S.level_start[1] = 1;
  }
  __syncwarp();
  int L = 0;
  for (;; ++L) {
    const uint32_t start = S.level_start[L], end = S.level_start[L + 1];
    uint32_t produced = 0;
    for (uint32_t base = start; base < end; base += 32) {
      const uint32_t i = base + lane;
      const bool valid = i < end;
      const uint32_t len = valid ? S.node_len[i] : 0;
      const bool internal = valid && len > (uint32_t)kNpBlock;
      const uint32_t m = __ballot_sync(0xffffffffu, internal);
      if (internal) {
        const uint32_t child = end + produced + 2 * __popc(m & ((1u << lane) - 1u));
        uint32_t h = len / 2;
        h -= h % 8;
        const uint32_t b = S.node_beg[i];
        S.node_beg[child] = b;
        S.node_len[child] = h;
        S.node_beg[child + 1] = b + h;
        S.node_len[child + 1] = len - h;
        S.node_child[i] = child;
      } else if (valid) {
        S.node_child[i] = kNpLeaf;
      }
      produced += 2 * __popc(m);
    }
    __syncwarp();
    if (produced == 0) break;
    if (lane == 0) S.level_start[L + 2] = end + produced;
    __syncwarp();
  }
  if (lane == 0) S.nlevels = L + 1;
}

// One term of numpy's sum, rounded like numpy: p = c / total (IEEE
// division), p * log2(p) (IEEE product) -- explicit _rn so nothing contracts.
__device__ __forceinline__ double np_term(double c, double total) {
  const double p = __ddiv_rn(c, total);
  return __dmul_rn(p, log2(p));
}

// terms[c] for c < nterms: either np_term(c, total) for c < kTermTable
// (term_table_kernel, one table per call: every pair of a judge call has the
// same total 2*H*W - 1), or a table the host registered for this total with
// pcbz_register_entropy_terms -- p * log2(p) evaluated by the host's own numpy
// for every count 0..total, so that every term, and with the emulated
// pairwise sum the entropy, has the reference's exact bits (numpy's SIMD
// log2 is not correctly rounded; the device's log2 differs from it in the
// last ulp for ~0.02 % of arguments).

// `get(bin)` returns the bin count (integer; 0 = empty); all NT threads of
// the block must call this.  `terms` may be null.
// If occ_ready, the caller has already filled S.occ (bit j of word w = bin
// 32w + j occupied) and synchronised.
template <int NT, typename Get>
__device__ double block_entropy_n(Get get, double total, NpScratchT<NT> &S, const double *terms,
                                  bool occ_ready = false, int64_t nterms = kTermTable,
                                  uint64_t *stamps = nullptr) {
  static_assert(NT % 32 == 0 && NT >= 64, "whole warps");
  const int t = threadIdx.x;
  auto stamp = [&](int i) {  // phase timestamps for profiling (PCBZ_TRACE_WORDS = 9)
    if (stamps && t == 0) {
      uint64_t v;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
      stamps[i] = v;
    }
  };
  // occupancy bitmap: one warp per 32-bin word (lane j reads bin 32w + j,
  // so the reads are bank-conflict free), a ballot makes the word
  if (!occ_ready) {
    // four words per warp step: their count reads are independent
    const int lane = t & 31;
    constexpr int kStep = NT / 32;
    for (int w0 = t >> 5; w0 < kOccWords; w0 += 4 * kStep) {
      bool occ[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int w = w0 + u * kStep;
        occ[u] = w < kOccWords && total > 0.0 && get(32 * w + lane) != 0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int w = w0 + u * kStep;
        const uint32_t bits = __ballot_sync(0xffffffffu, occ[u]);
        if (lane == 0 && w < kOccWords) S.occ[w] = bits;
      }
    }
  }
  __syncthreads();
  stamp(0);
  const int w_lo = occ_word_lo<NT>(t), w_hi = occ_word_lo<NT>(t + 1);
  uint32_t cnt = 0;
  for (int w = w_lo; w < w_hi; ++w) cnt += __popc(S.occ[w]);
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if ((t & 31) >= o) incl += v;
  }
  __syncthreads();
  if ((t & 31) == 31) S.off[t >> 5] = incl;  // warp totals, temporarily
  __syncthreads();
  uint32_t base = 0, n_all = 0;
  for (int w = 0; w < NT / 32; ++w) {
    const uint32_t v = S.off[w];
    if (w < (t >> 5)) base += v;
    n_all += v;
  }
  __syncthreads();
  S.off[t] = base + incl - cnt;
  if (t == 0) S.off[NT] = n_all;
  if (n_all == 0 || !(total > 0.0)) {
    __syncthreads();
    return 0.0;
  }
  stamp(1);
  if (t < 32) np_build_tree(n_all, S);
  __syncthreads();
  stamp(2);
  const int nodes = (int)S.level_start[S.nlevels];
  // a host-registered table covers every count (nterms = total + 1)
  const bool full_table = terms && (double)nterms > total;
  auto term_of = [&](uint64_t c) -> double {
    if (full_table) return __ldg(terms + c);
    if (!terms) return np_term((double)c, total);
    const bool in = c < (uint64_t)nterms;
    const double v = __ldg(terms + (in ? c : 0));
    return in ? v : np_term((double)c, total);
  };
  // ---- leaves ---------------------------------------------------------------
  for (int j = t; j < nodes; j += NT) {
    if (S.node_child[j] != kNpLeaf) continue;
    const uint32_t beg = S.node_beg[j], len = S.node_len[j];
    int r0 = 0, r1 = NT - 1;  // last thread range with off <= beg
    while (r0 < r1) {
      const int mid = (r0 + r1 + 1) >> 1;
      if (S.off[mid] <= beg) r0 = mid; else r1 = mid - 1;
    }
    int w = occ_word_lo<NT>(r0);
    uint32_t idx = S.off[r0];
    uint32_t bits = S.occ[w];
    while (idx + __popc(bits) <= beg) {
      idx += __popc(bits);
      bits = S.occ[++w];
    }
    for (uint32_t k = beg - idx; k > 0; --k) bits &= bits - 1;  // drop earlier terms
    auto next_bin = [&]() -> int {
      while (!bits) bits = S.occ[++w];
      const int bin = 32 * w + __ffs(bits) - 1;
      bits &= bits - 1;
      return bin;
    };
    auto next_term = [&]() -> double { return term_of(get(next_bin())); };
    // eight terms at a time: bin indices first (bitmap walk), then all eight
    // count reads and table loads in flight together
    auto next8 = [&](double (&v)[8]) {
      int b[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) b[q] = next_bin();
      uint64_t c[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) c[q] = get(b[q]);
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = term_of(c[q]);
    };
    double res;
    if (len < 8) {
      res = -0.0;
      for (uint32_t i = 0; i < len; ++i) res = __dadd_rn(res, next_term());
    } else {
      double r[8];
      next8(r);
      uint32_t i = 8;
      for (; i < len - (len % 8); i += 8) {
        double v[8];
        next8(v);
#pragma unroll
        for (int q = 0; q < 8; ++q) r[q] = __dadd_rn(r[q], v[q]);
      }
      res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                      __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
      for (; i < len; ++i) res = __dadd_rn(res, next_term());
    }
    S.node_sum[j] = res;
  }
  __syncthreads();
  stamp(3);
  // ---- internal nodes, deepest level first ----------------------------------
  for (int L = S.nlevels - 2; L >= 0; --L) {
    for (int j = (int)S.level_start[L] + t; j < (int)S.level_start[L + 1]; j += NT) {
      const uint32_t c = S.node_child[j];
      if (c != kNpLeaf) S.node_sum[j] = __dadd_rn(S.node_sum[c], S.node_sum[c + 1]);
    }
    __syncthreads();
  }
  const double e = -S.node_sum[0];
  __syncthreads();
  return e;
}

// the judge kernel's shape (kEntropyThreads)
template <typename Get>
__device__ __forceinline__ double block_entropy(Get get, double total, NpScratch &S, const double *terms,
                                                bool occ_ready = false, int64_t nterms = kTermTable,
                                                uint64_t *stamps = nullptr) {
  return block_entropy_n<kEntropyThreads>(get, total, S, terms, occ_ready, nterms, stamps);
}

}  // namespace pcbz
