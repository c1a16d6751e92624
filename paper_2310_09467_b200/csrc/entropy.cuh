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
// _core/src/umath/loops_utils.h.src; checked bit-for-bit against np.sum for
// n = 1..65536 in tests/test_entropy_emulation.py).  Every term is rounded
// exactly like numpy's (IEEE division, device log2, IEEE product), so the
// device entropy equals the reference's whenever log2 rounds alike (both
// are correctly rounded for nearly all arguments), and mathematically tied
// candidates tie or break exactly as in the reference.
//
// Parallel form: thread t owns a run of 32-bin occupancy words; a block
// scan of occupied counts gives every occupied bin its index in the
// (virtual) compacted term array; the recursion's leaves -- index ranges of
// at most 128 terms -- are evaluated by different threads walking the
// occupancy bitmap; thread 0 folds the leaf sums in recursion order.
#pragma once
#include <cstdint>

#include "judge.cuh"

namespace pcbz {

constexpr int kNpLeafMax = 1024;  // leaves hold >= 64 terms once n > 128
constexpr int kNpBlock = 128;     // numpy PW_BLOCKSIZE
constexpr int kOccWords = 2048;   // 65536 bins / 32

struct NpScratch {
  uint32_t off[kEntropyThreads + 1];  // compacted index of each thread's first term
  uint32_t occ[kOccWords];            // occupancy bitmap
  uint32_t leaf_beg[kNpLeafMax];
  uint32_t leaf_len[kNpLeafMax];
  double leaf_sum[kNpLeafMax];
  double result;
  int nleaf;
};

__device__ __forceinline__ int occ_word_lo(int t) { return (kOccWords * t) / kEntropyThreads; }

// leaves of numpy's pairwise recursion over n terms, in left-to-right order
__device__ inline void np_enumerate_leaves(uint32_t n, NpScratch &S) {
  uint32_t st_b[48], st_n[48];
  int sp = 0, nl = 0;
  st_b[sp] = 0; st_n[sp] = n; ++sp;
  while (sp) {
    --sp;
    const uint32_t b = st_b[sp], m = st_n[sp];
    if (m <= (uint32_t)kNpBlock) {
      S.leaf_beg[nl] = b; S.leaf_len[nl] = m; ++nl;
    } else {
      uint32_t h = m / 2;
      h -= h % 8;
      st_b[sp] = b + h; st_n[sp] = m - h; ++sp;  // right half is popped after the left
      st_b[sp] = b; st_n[sp] = h; ++sp;
    }
  }
  S.nleaf = nl;
}

// pairwise(a, n) = pairwise(left) + pairwise(right), from the leaf sums
__device__ inline double np_fold(uint32_t n, const NpScratch &S) {
  uint32_t st_n[48];
  uint8_t st_state[48];
  double st_left[48];
  int sp = 1, leaf = 0;
  double ret = 0.0;
  st_n[0] = n; st_state[0] = 0;
  while (sp) {
    const int top = sp - 1;
    const uint32_t m = st_n[top];
    if (m <= (uint32_t)kNpBlock) {
      ret = S.leaf_sum[leaf++];
      --sp;
      continue;
    }
    uint32_t h = m / 2;
    h -= h % 8;
    if (st_state[top] == 0) {
      st_state[top] = 1;
      st_n[sp] = h; st_state[sp] = 0; ++sp;
    } else if (st_state[top] == 1) {
      st_left[top] = ret;
      st_state[top] = 2;
      st_n[sp] = m - h; st_state[sp] = 0; ++sp;
    } else {
      ret = st_left[top] + ret;
      --sp;
    }
  }
  return ret;
}

// `get(bin)` returns the bin count as a double (0 = empty); all threads of
// the block (kEntropyThreads) must call this.
template <typename Get>
__device__ double block_entropy(Get get, double total, NpScratch &S) {
  const int t = threadIdx.x;
  const int w_lo = occ_word_lo(t), w_hi = occ_word_lo(t + 1);
  uint32_t cnt = 0;
  for (int w = w_lo; w < w_hi; ++w) {
    uint32_t bits = 0;
    if (total > 0.0) {
#pragma unroll 8
      for (int j = 0; j < 32; ++j) bits |= (get(32 * w + j) > 0.0 ? 1u : 0u) << j;
    }
    S.occ[w] = bits;
    cnt += __popc(bits);
  }
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
  for (int w = 0; w < kEntropyThreads / 32; ++w) {
    const uint32_t v = S.off[w];
    if (w < (t >> 5)) base += v;
    n_all += v;
  }
  __syncthreads();
  S.off[t] = base + incl - cnt;
  if (t == 0) {
    S.off[kEntropyThreads] = n_all;
    if (n_all > 0) np_enumerate_leaves(n_all, S);
    else S.nleaf = 0;
  }
  __syncthreads();
  const int nleaf = S.nleaf;
  for (int L = t; L < nleaf; L += kEntropyThreads) {
    const uint32_t beg = S.leaf_beg[L], len = S.leaf_len[L];
    int r0 = 0, r1 = kEntropyThreads - 1;  // last thread range with off <= beg
    while (r0 < r1) {
      const int mid = (r0 + r1 + 1) >> 1;
      if (S.off[mid] <= beg) r0 = mid; else r1 = mid - 1;
    }
    int w = occ_word_lo(r0);
    uint32_t idx = S.off[r0];
    uint32_t bits = S.occ[w];
    while (idx + __popc(bits) <= beg) {
      idx += __popc(bits);
      bits = S.occ[++w];
    }
    for (uint32_t k = beg - idx; k > 0; --k) bits &= bits - 1;  // drop earlier terms
    auto next_term = [&]() -> double {
      while (!bits) bits = S.occ[++w];
      const int bin = 32 * w + __ffs(bits) - 1;
      bits &= bits - 1;
      // explicit IEEE ops: no FMA contraction may fuse the product into the
      // running sum (numpy rounds p*log2(p) before summing)
      const double p = __ddiv_rn(get(bin), total);
      return __dmul_rn(p, log2(p));
    };
    double res;
    if (len < 8) {
      res = -0.0;
      for (uint32_t i = 0; i < len; ++i) res = __dadd_rn(res, next_term());
    } else {
      double r[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = next_term();
      uint32_t i = 8;
      for (; i < len - (len % 8); i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], next_term());
      }
      res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
      for (; i < len; ++i) res = __dadd_rn(res, next_term());
    }
    S.leaf_sum[L] = res;
  }
  __syncthreads();
  if (t == 0) S.result = (total > 0.0 && n_all > 0) ? -np_fold(n_all, S) : 0.0;
  __syncthreads();
  const double e = S.result;
  __syncthreads();
  return e;
}

}  // namespace pcbz
