// bzip2.cu -- libbzip2 1.0.8 level-9 block coder on the GPU, byte-exact with
// bz2.compress(chunk, 9): the back end the reference runs on host threads
// (pkg/src/pcbz/blocks.py:73-81 -> stdlib bz2 -> libbz2 1.0.8, SURVEY §8(f)
// rank 4).  The algorithm is restated in oracle/bzip2_ref.py (pinned against
// libbz2 by tests/test_bzip2_ref.py); stages follow it.
//
// Many independent inputs ("jobs", one per PCBZ block) are coded together:
//   A  RLE1              runs -> 255-byte chunk events -> output offsets
//                        (scan), libbz2's greedy block split (binary search
//                        per job), bytes, block CRCs (GF(2)-linear, chunked),
//                        used-symbol maps
//   B  prefix doubling   cyclic-rotation sort of every block at once: radix
//                        sorts (radix_sort.cuh) of (group, partner rank) keys
//                        over the shrinking set of unresolved groups
//   C  mtf_kernel        one thread per block: BWT column, MTF, RUNA/RUNB
//   D  tables_kernel     one CTA per block: initial tables, four refinement
//                        passes (parallel over 50-symbol groups), huffman.c
//                        code lengths, selector MTF, bit counts
//   E  emit_kernel       one CTA per block: header fields, then every code at
//                        its scanned bit offset (atomicOr into the job's
//                        big-endian word stream); frame_kernel adds 'BZh9'
//                        and the end-of-stream marker + combined CRC
// A block whose rotations tie (an exactly periodic block) flags its job for
// the host libbz2: libbz2 orders equal rotations by its quicksort
// refinements, which are not restated.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/pcbz_b200.h"
#include "radix_sort.cuh"

namespace pcbz {
namespace bz {

constexpr int kBlockMax = 899981;          // 100000 * 9 - 19 (bzlib.c nblockMAX)
constexpr int kMaxAlpha = 258;
constexpr int kMaxGroups = 6;
constexpr int kGroupSize = 50;
constexpr int kMaxCodeLen = 17;
constexpr int kTableThreads = 256;
constexpr int kEmitThreads = 256;
constexpr int kEmitItems = 8;

struct Job {
  int64_t in_off, in_len;
  int64_t rle_off;        // RLE1 output region
  int32_t block0;         // first block slot
  int32_t nblocks;        // filled by stage A
};

struct Block {
  int64_t rle_off;        // absolute offset of the block's bytes in the RLE buffer
  int32_t n;              // block bytes
  int32_t job;
  uint32_t crc;
  uint32_t in_use[8];
  uint32_t base;          // first global element index (stage B)
  int32_t orig, tie;
  int64_t mtf_off;        // into mtfv (room for n + 1 values)
  int64_t sel_off;        // into selectors (room for (n + 1 + 49) / 50)
  int32_t n_mtf, n_groups, n_sel, n_in_use;
  int64_t hdr_bits, data_bits;
  int64_t bit_off;        // absolute bit position in the output word stream
  uint32_t in_begin, in_end;   // the job input bytes this block codes (stage A)
};

__device__ __forceinline__ uint32_t crc_entry(uint32_t i) {
  uint32_t c = i << 24;
  for (int k = 0; k < 8; ++k) c = (c & 0x80000000u) ? (c << 1) ^ 0x04C11DB7u : (c << 1);
  return c;
}

// ---------------------------------------------------------------------------
// A: RLE1 + block split (bzlib.c ADD_CHAR_TO_BLOCK, add_pair_to_block,
// copy_input_until_stop, handle_compress as driven by bz2.compress)
// ---------------------------------------------------------------------------

// Stage A in parallel (oracle/bzip2_ref.py rle1_blocks is the sequential
// restatement):
//   runs       maximal runs of one byte value (job starts force a run start)
//   events     a run of L bytes is added as floor(L/255) chunks of 255 (5
//              output bytes: 4 x ch + 251) and a remainder r (r <= 3: r bytes,
//              else 5) -- bzlib.c flushes a run at 255 and at its end
//   blocks     greedy over events: a block closes after the first event that
//              brings it to >= nblockMAX bytes (the check before every input
//              char), so a block may end inside a long run
//   CRC        linear over GF(2): each 4 KB chunk's CRC from a zero register,
//              shifted by the bytes after it in the block (32x32 bit-matrix
//              powers of "append a zero byte"), XORed together with the
//              shifted initial register

__constant__ uint32_t c_zero_shift[32][32];   // [k][bit]: image of bit after 2^k zero bytes

__device__ __forceinline__ uint32_t gf2_apply(int k, uint32_t v) {
  uint32_t r = 0;
#pragma unroll 4
  for (int b = 0; b < 32; ++b)
    if (v & (1u << b)) r ^= c_zero_shift[k][b];
  return r;
}

__device__ uint32_t crc_shift(uint32_t v, uint64_t nbytes) {
  for (int k = 0; nbytes; ++k, nbytes >>= 1)
    if (nbytes & 1) v = gf2_apply(k, v);
  return v;
}

__device__ __forceinline__ uint32_t run_out_bytes(uint32_t L) {
  const uint32_t rem = L % 255;
  return 5 * (L / 255) + (rem <= 3 ? rem : 5);
}

__global__ void run_flags_kernel(const uint8_t *in, int64_t total, uint8_t *flags) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = (i == 0 || in[i] != in[i - 1]) ? 1 : 0;
}

__global__ void job_start_flags_kernel(const int64_t *in_off, int njobs, uint8_t *flags) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < njobs && in_off[j] < in_off[j + 1]) flags[in_off[j]] = 1;
}

__global__ void iota64_kernel(uint32_t *a, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (uint32_t)i;
}

__global__ void run_sizes_kernel(const uint32_t *rs, uint32_t R, uint32_t total, uint32_t *osz) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += gridDim.x * blockDim.x) {
    const uint32_t e = r + 1 < R ? rs[r + 1] : total;
    osz[r] = run_out_bytes(e - rs[r]);
  }
}

// one thread per job: block split by binary search over the runs' output
// offsets (ocum: exclusive scan of the run sizes, R + 1 entries)
__global__ void split_kernel(const int64_t *in_off, int njobs, const uint32_t *rs, uint32_t R,
                             uint32_t total, const uint32_t *ocum, Job *jobs, Block *blocks) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= njobs) return;
  Job &J = jobs[j];
  J.nblocks = 0;
  if (in_off[j] == in_off[j + 1]) return;
  auto lower = [&](uint32_t x) {  // first run with rs >= x
    uint32_t lo = 0, hi = R;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (rs[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  const uint32_t r0 = lower((uint32_t)in_off[j]), r1 = lower((uint32_t)in_off[j + 1]);
  auto run_end = [&](uint32_t r) { return r + 1 < R ? rs[r + 1] : total; };
  uint32_t start = ocum[r0];
  const uint32_t end = ocum[r1];
  uint32_t in_start = rs[r0];
  uint32_t r = r0;
  int nb = 0;
  while (start < end) {
    uint32_t bend, in_end;
    if (end - start < (uint32_t)kBlockMax) {
      bend = end;
      in_end = (uint32_t)in_off[j + 1];
    } else {
      // first run rr >= r whose end brings the block to >= kBlockMax
      uint32_t lo = r, hi = r1 - 1;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (ocum[mid + 1] - start >= (uint32_t)kBlockMax) hi = mid; else lo = mid + 1;
      }
      const uint32_t rr = lo;
      const int64_t c0 = (int64_t)ocum[rr] - (int64_t)start;   // may be < 0 mid-run
      const uint32_t L = run_end(rr) - rs[rr];
      const int64_t nfull = L / 255;
      const int64_t e = (kBlockMax - c0 + 4) / 5;                // chunk events needed
      if (nfull > 0 && e <= nfull) {
        bend = ocum[rr] + (uint32_t)(5 * e);
        in_end = rs[rr] + (uint32_t)(255 * e);
        r = rr;
      } else {
        bend = ocum[rr + 1];
        in_end = run_end(rr);
        r = rr + 1;
      }
    }
    Block &B = blocks[J.block0 + nb];
    B.rle_off = start;
    B.n = (int32_t)(bend - start);
    B.job = j;
    B.tie = 0;
    B.in_begin = in_start;
    B.in_end = in_end;
    ++nb;
    start = bend;
    in_start = in_end;
  }
  J.nblocks = nb;
}

__global__ void run_write_kernel(const uint8_t *in, const uint32_t *rs, uint32_t R, uint32_t total,
                                 const uint32_t *ocum, uint8_t *rle) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += gridDim.x * blockDim.x) {
    const uint32_t b = rs[r], L = (r + 1 < R ? rs[r + 1] : total) - b;
    const uint8_t ch = in[b];
    uint8_t *o = rle + ocum[r];
    for (uint32_t k = 0; k < L / 255; ++k) {
      o[0] = o[1] = o[2] = o[3] = ch;
      o[4] = 251;
      o += 5;
    }
    const uint32_t rem = L % 255;
    if (rem <= 3) {
      for (uint32_t k = 0; k < rem; ++k) o[k] = ch;
    } else {
      o[0] = o[1] = o[2] = o[3] = ch;
      o[4] = (uint8_t)(rem - 4);
    }
  }
}

constexpr int kCrcChunk = 4096;

// grid: (chunk, block) pairs; acc[b] ^= shifted CRC of one input chunk
__global__ void crc_chunks_kernel(const uint8_t *in, const Block *blocks, const int *ids,
                                  const uint32_t *chunk0, int nb, uint32_t *acc) {
  __shared__ uint32_t tab[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) tab[i] = crc_entry(i);
  __syncthreads();
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  // block of chunk c: last t with chunk0[t] <= c
  int lo = 0, hi = nb;  // chunk0 has nb + 1 entries
  if (c >= chunk0[nb]) return;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (chunk0[mid] <= c) lo = mid; else hi = mid;
  }
  const Block &B = blocks[ids[lo]];
  const uint32_t ib = B.in_begin, ie = B.in_end;
  const uint32_t a = ib + (c - chunk0[lo]) * kCrcChunk;
  const uint32_t e = min(ie, a + kCrcChunk);
  uint32_t crc = 0;
  for (uint32_t i = a; i < e; ++i) crc = (crc << 8) ^ tab[(crc >> 24) ^ in[i]];
  crc = crc_shift(crc, ie - e);
  if (c == chunk0[lo]) crc ^= crc_shift(0xFFFFFFFFu, ie - ib);   // the initial register
  atomicXor(&acc[lo], crc);
}

// one CTA per block: final CRC and the used-byte map of its RLE1 bytes
__global__ void block_meta_kernel(const uint8_t *rle, Block *blocks, const int *ids, const uint32_t *acc) {
  __shared__ uint8_t seen[256];
  Block &B = blocks[ids[blockIdx.x]];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) seen[i] = 0;
  __syncthreads();
  const uint8_t *d = rle + B.rle_off;
  for (int i = threadIdx.x; i < B.n; i += blockDim.x) seen[d[i]] = 1;
  __syncthreads();
  if (threadIdx.x < 8) {
    uint32_t w = 0;
    for (int b = 0; b < 32; ++b) w |= (uint32_t)seen[32 * threadIdx.x + b] << b;
    B.in_use[threadIdx.x] = w;
  }
  if (threadIdx.x == 0) B.crc = ~acc[blockIdx.x];
}

// ---------------------------------------------------------------------------
// B: cyclic rotation sort by prefix doubling
// ---------------------------------------------------------------------------

__global__ void fill_block_of_kernel(const Block *blocks, const int *ids, uint32_t *block_of) {
  const Block &B = blocks[ids[blockIdx.x]];
  for (int i = threadIdx.x; i < B.n; i += blockDim.x) block_of[B.base + i] = (uint32_t)ids[blockIdx.x];
}

__global__ void init_keys_kernel(const Block *blocks, const uint32_t *block_of, const uint8_t *rle,
                                 uint32_t N, uint64_t *keys, uint32_t *vals) {
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < N; g += gridDim.x * blockDim.x) {
    const uint32_t b = block_of[g];
    const Block &B = blocks[b];
    const uint32_t i = g - B.base, n = (uint32_t)B.n;
    const uint8_t *d = rle + B.rle_off;
    uint32_t k = 0;
    for (int t = 0; t < 4; ++t) k = (k << 8) | d[(i + t) % n];
    keys[g] = ((uint64_t)b << 32) | k;
    vals[g] = g;
  }
}

__global__ void heads_kernel(const uint64_t *keys, uint32_t m, uint8_t *hd) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x)
    hd[k] = (k == 0 || keys[k] != keys[k - 1]) ? 1 : 0;
}

// gs[k] = (hd[k] ? pos(k) : 0), pos = U[k] (or k for the first round)
__global__ void head_pos_kernel(const uint8_t *hd, const uint32_t *U, uint32_t m, uint32_t *gs) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x)
    gs[k] = hd[k] ? (U ? U[k] : k) : 0u;
}

struct MaxOp {
  __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return a > b ? a : b; }
};

// after a sort of m elements (sorted vals, their slots U[k] or k): write the
// suffix array, the new ranks and the unresolved flags; groups of blocks
// whose compared prefix (plen) already covers the whole block are ties
__global__ void settle_kernel(const uint32_t *vals, const uint32_t *U, uint32_t m, const uint8_t *hd,
                              const uint32_t *gs, uint32_t *sa, uint32_t *rank, const uint32_t *block_of,
                              Block *blocks, uint64_t plen, uint8_t *unres) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x) {
    const uint32_t g = vals[k];
    const uint32_t slot = U ? U[k] : k;
    sa[slot] = g;
    rank[g] = gs[k];
    const bool open = !hd[k] || (k + 1 < m && !hd[k + 1]);
    uint8_t u = 0;
    if (open) {
      // a block's suffix-array slots are its own position range [base, base
      // + n) (the first sort orders by block id, ids ascend with base), so
      // the slot's block is g's block: a sequential read, not a random one
      const uint32_t b = block_of[slot];
      if (plen >= (uint64_t)blocks[b].n) blocks[b].tie = 1;  // equal full rotations
      else u = 1;
    }
    unres[k] = u;
  }
}

__global__ void pair_keys_kernel(const uint32_t *U, uint32_t m, const uint32_t *sa, const uint32_t *rank,
                                 const uint32_t *block_of, const Block *blocks, uint64_t h,
                                 uint64_t *keys, uint32_t *vals) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x) {
    const uint32_t g = sa[U[k]];
    const Block &B = blocks[block_of[g]];
    const uint32_t n = (uint32_t)B.n;
    const uint32_t p = B.base + (uint32_t)(((uint64_t)(g - B.base) + h) % n);
    keys[k] = ((uint64_t)rank[g] << 32) | rank[p];
    vals[k] = g;
  }
}

// ---------------------------------------------------------------------------
// C: BWT column, MTF and zero-run coding (compress.c generateMTFValues)
// ---------------------------------------------------------------------------
//
// One warp per segment of a block's BWT column (C3 below); BWT characters
// are gathered 32 at a time.

constexpr int kMtfWarps = 4;

// Segment-parallel form: the MTF list at any position is "symbols by most
// recent occurrence, then the never-seen ones in symbol order", so each
// segment of kMtfSeg symbols starts from a list built out of the last
// occurrences before it (a prefix max over the block's segments) and runs
// on its own warp, emitting ranks.  Zero-run coding is then vectorised: a
// nonzero rank knows the zero run before it from a max-scan of nonzero
// positions, its output count (bijective base-2 digits + 1) is scanned into
// offsets, and every position writes its own symbols.

constexpr int kMtfSeg = 8192;

__device__ __forceinline__ int find_seg(const uint32_t *seg0, int nb, uint32_t s) {
  int lo = 0, hi = nb;  // seg0 has nb + 1 entries; last t with seg0[t] <= s
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (seg0[mid] <= s) lo = mid; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ void symbol_map(const Block &B, uint8_t *u2s, int lane, int &nin) {
  nin = 0;
  for (int base = 0; base < 256; base += 32) {
    const int c = base + lane;
    const bool used = (B.in_use[c >> 5] >> (c & 31)) & 1u;
    const uint32_t m = __ballot_sync(0xffffffffu, used);
    if (used) u2s[c] = (uint8_t)(nin + __popc(m & ((1u << lane) - 1u)));
    nin += __popc(m);
  }
  __syncwarp();
}

// C1: BWT column as symbols (makeMaps_e numbering), last occurrence of every
// symbol per segment, origPtr
__global__ void __launch_bounds__(32 * kMtfWarps) mtf_gather_kernel(Block *blocks, const int *ids, int nb,
                                                                     const uint32_t *seg0, const uint32_t *sa,
                                                                     const uint8_t *rle, uint8_t *symseq,
                                                                     int32_t *lastpos) {
  __shared__ uint8_t s_u2s[kMtfWarps][256];
  __shared__ int32_t s_last[kMtfWarps][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t sg = blockIdx.x * kMtfWarps + warp;
  if (sg >= seg0[nb]) return;
  const int t = find_seg(seg0, nb, sg);
  Block &B = blocks[ids[t]];
  const uint32_t k = sg - seg0[t];
  uint8_t *u2s = s_u2s[warp];
  int32_t *last = s_last[warp];
  int nin;
  symbol_map(B, u2s, lane, nin);
  if (k == 0 && lane == 0) B.n_in_use = nin;
  for (int x = lane; x < 256; x += 32) last[x] = -1;
  __syncwarp();
  const uint32_t n = (uint32_t)B.n;
  const uint32_t j0 = k * kMtfSeg, j1 = min(n, j0 + kMtfSeg);
  const uint8_t *d = rle + B.rle_off;
  for (uint32_t j = j0 + lane; j < j1; j += 32) {
    const uint32_t i = sa[B.base + j] - B.base;
    if (i == 0) B.orig = (int32_t)j;
    const uint8_t sym = u2s[d[i == 0 ? n - 1 : i - 1]];
    symseq[B.base + j] = sym;
    atomicMax(&last[sym], (int32_t)j);
  }
  __syncwarp();
  for (int x = lane; x < 256; x += 32) lastpos[(size_t)sg * 256 + x] = last[x];
}

// C2: last occurrence before each segment (one CTA of 256 per block)
__global__ void mtf_prefix_kernel(const uint32_t *seg0, int32_t *lastpos) {
  const int x = threadIdx.x;
  int32_t run = -1;
  for (uint32_t sg = seg0[blockIdx.x]; sg < seg0[blockIdx.x + 1]; ++sg) {
    const int32_t v = lastpos[(size_t)sg * 256 + x];
    lastpos[(size_t)sg * 256 + x] = run;   // now: last occurrence BEFORE the segment
    run = max(run, v);
  }
}

// C3: MTF ranks of one segment (warp).  The warp holds the inverse of the
// MTF list -- the current position of every symbol -- as 16-bit fields, lane
// l owning symbols 8l..8l+7 in four registers.  Coding symbol s: its owner's
// field is the rank r (one byte permute + one shuffle); every symbol at a
// position below r moves down one (SWAR: the borrow of (b | 0x8000) - r in
// each field's guard bit), and s itself goes to position 0.  About 35
// instructions per symbol with no data-dependent branch, against ~75 for a
// list kept in list order (find by byte compare + ballot, shift by a
// shuffled carry byte), measured 77 ms on C2 (profiles/r01_compress_launches_c2_100.txt).
__global__ void __launch_bounds__(32 * kMtfWarps) mtf_rank_kernel(const Block *blocks, const int *ids, int nb,
                                                                   const uint32_t *seg0, const uint8_t *symseq,
                                                                   const int32_t *before, uint8_t *ranks) {
  __shared__ int32_t s_bef[kMtfWarps][256];
  __shared__ uint8_t s_at[kMtfWarps][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t sg = blockIdx.x * kMtfWarps + warp;
  if (sg >= seg0[nb]) return;
  const int t = find_seg(seg0, nb, sg);
  const Block &B = blocks[ids[t]];
  const uint32_t k = sg - seg0[t];
  int32_t *bef = s_bef[warp];
  uint8_t *at = s_at[warp];   // at[symbol] = its position in the segment's initial list
  int seen_mine = 0;
  for (int x = lane; x < 256; x += 32) {
    bef[x] = before[(size_t)sg * 256 + x];
    seen_mine += bef[x] >= 0;
  }
  int nseen = seen_mine;
  for (int o = 16; o > 0; o >>= 1) nseen += __shfl_xor_sync(0xffffffffu, nseen, o);
  __syncwarp();
  for (int x = lane; x < 256; x += 32) {  // initial list position of symbol x
    const int32_t bx = bef[x];
    int pos = 0;
    if (bx >= 0) {
      for (int y = 0; y < 256; ++y) pos += bef[y] > bx;
    } else {
      pos = nseen;
      for (int y = 0; y < x; ++y) pos += bef[y] < 0;
    }
    at[x] = (uint8_t)pos;
  }
  __syncwarp();
  uint32_t w0, w1, w2, w3;   // positions of symbols 8l + {0,1}, {2,3}, {4,5}, {6,7}
  w0 = at[8 * lane + 0] | ((uint32_t)at[8 * lane + 1] << 16);
  w1 = at[8 * lane + 2] | ((uint32_t)at[8 * lane + 3] << 16);
  w2 = at[8 * lane + 4] | ((uint32_t)at[8 * lane + 5] << 16);
  w3 = at[8 * lane + 6] | ((uint32_t)at[8 * lane + 7] << 16);
  const uint32_t n = (uint32_t)B.n;
  const uint32_t j0 = k * kMtfSeg, j1 = min(n, j0 + kMtfSeg);
  for (uint32_t jb = j0; jb < j1; jb += 32) {
    const uint32_t j = jb + lane;
    const uint32_t sym = j < j1 ? symseq[B.base + j] : 0u;
    const int cnt = (int)min(32u, j1 - jb);
    uint32_t myrank = 0;
    for (int q = 0; q < cnt; ++q) {
      const uint32_t s = __shfl_sync(0xffffffffu, sym, q);
      const uint32_t f = s & 7u;                      // field of s in its owner lane
      const uint32_t lo = f & 4u ? w2 : w0, hi = f & 4u ? w3 : w1;
      const uint32_t b0 = (f & 3u) * 2u;              // its two bytes within (hi:lo)
      const uint32_t mine = __byte_perm(lo, hi, b0 | ((b0 + 1u) << 4)) & 0xFFFFu;
      const uint32_t r = __shfl_sync(0xffffffffu, mine, (int)(s >> 3));
      const uint32_t R2 = r * 0x00010001u;
      // fields b < r gain one: no borrow into the guard bit of (b | 0x8000) - r
      w0 += (~(w0 + 0x80008000u - R2) & 0x80008000u) >> 15;
      w1 += (~(w1 + 0x80008000u - R2) & 0x80008000u) >> 15;
      w2 += (~(w2 + 0x80008000u - R2) & 0x80008000u) >> 15;
      w3 += (~(w3 + 0x80008000u - R2) & 0x80008000u) >> 15;
      // s (field value r, unchanged above) moves to the front
      const uint32_t clr = lane == (int)(s >> 3) ? r << ((f & 1u) << 4) : 0u;
      const uint32_t wi = f >> 1;
      w0 -= wi == 0u ? clr : 0u;
      w1 -= wi == 1u ? clr : 0u;
      w2 -= wi == 2u ? clr : 0u;
      w3 -= wi == 3u ? clr : 0u;
      myrank = lane == q ? r : myrank;
    }
    if (j < j1) ranks[B.base + j] = (uint8_t)myrank;
  }
}

__device__ __forceinline__ uint32_t run_digits(uint32_t L) { return L ? 31u - __clz(L + 1u) : 0u; }

// C4: zero-run coding
__global__ void nz_pos_kernel(const uint8_t *ranks, uint32_t N, uint32_t *P) {
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < N; g += gridDim.x * blockDim.x)
    P[g] = ranks[g] ? g + 1 : 0u;
}

__device__ __forceinline__ uint32_t zeros_before(const uint32_t *P, uint32_t g, uint32_t base) {
  // zero ranks strictly between the previous nonzero rank of the block (or
  // its start) and g
  const uint32_t pp = g > base ? P[g - 1] : 0u;
  const int64_t prev = pp > base ? (int64_t)pp - 1 : (int64_t)base - 1;
  return (uint32_t)((int64_t)g - prev - 1);
}

__global__ void run_count_kernel(const uint8_t *ranks, const uint32_t *P, const uint32_t *block_of,
                                 const Block *blocks, uint32_t N, uint32_t *cnt) {
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g <= N; g += gridDim.x * blockDim.x) {
    if (g == N) { cnt[g] = 0; continue; }
    if (!ranks[g]) { cnt[g] = 0; continue; }
    const uint32_t base = blocks[block_of[g]].base;
    cnt[g] = run_digits(zeros_before(P, g, base)) + 1;
  }
}

__device__ __forceinline__ uint16_t *put_run(uint16_t *o, uint32_t L) {
  if (!L) return o;
  uint32_t z = L - 1;
  for (;;) {
    *o++ = (z & 1) ? 1 : 0;  // RUNB : RUNA
    if (z < 2) break;
    z = (z - 2) / 2;
  }
  return o;
}

__global__ void run_write_mtf_kernel(const uint8_t *ranks, const uint32_t *P, const uint32_t *off,
                                     const uint32_t *block_of, const Block *blocks, uint32_t N,
                                     uint16_t *mtfv) {
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < N; g += gridDim.x * blockDim.x) {
    const uint32_t r = ranks[g];
    if (!r) continue;
    const Block &B = blocks[block_of[g]];
    uint16_t *o = mtfv + B.mtf_off + (off[g] - off[B.base]);
    o = put_run(o, zeros_before(P, g, B.base));
    *o = (uint16_t)(r + 1);
  }
}

// tail (zero run before EOB, EOB) and symbol frequencies: one CTA per block
__global__ void mtf_tail_freq_kernel(Block *blocks, const int *ids, const uint32_t *P, const uint32_t *off,
                                     uint16_t *mtfv, uint32_t *freq_out) {
  __shared__ uint32_t hist[8][kMaxAlpha];
  __shared__ int32_t s_nmtf;
  Block &B = blocks[ids[blockIdx.x]];
  if (B.tie) return;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 8 * kMaxAlpha; i += blockDim.x) (&hist[0][0])[i] = 0;
  if (threadIdx.x == 0) {
    const uint32_t last = B.base + (uint32_t)B.n - 1;
    const uint32_t pp = P[last];
    const int64_t prev = pp > B.base ? (int64_t)pp - 1 : (int64_t)B.base - 1;
    const uint32_t L = (uint32_t)((int64_t)last - prev);
    const uint32_t w = off[B.base + B.n] - off[B.base];
    uint16_t *o = put_run(mtfv + B.mtf_off + w, L);
    *o = (uint16_t)(B.n_in_use + 1);     // EOB
    s_nmtf = (int32_t)(o + 1 - (mtfv + B.mtf_off));
  }
  __syncthreads();
  const int n_mtf = s_nmtf;
  const uint16_t *mv = mtfv + B.mtf_off;
  for (int i = threadIdx.x; i < n_mtf; i += blockDim.x) atomicAdd(&hist[warp][mv[i]], 1u);
  __syncthreads();
  for (int v = threadIdx.x; v < kMaxAlpha; v += blockDim.x) {
    uint32_t c = 0;
    for (int w = 0; w < 8; ++w) c += hist[w][v];
    freq_out[(size_t)ids[blockIdx.x] * kMaxAlpha + v] = c;
  }
  if (threadIdx.x == 0) B.n_mtf = n_mtf;
}

// ---------------------------------------------------------------------------
// D: coding tables (compress.c sendMTFValues, huffman.c)
// ---------------------------------------------------------------------------

// BZ2_hbMakeCodeLengths, heap operations and tie-breaks as in huffman.c
struct HuffWork {   // BZ2_hbMakeCodeLengths work arrays (shared memory, one per table)
  int32_t heap[kMaxAlpha + 2];
  int32_t weight[kMaxAlpha * 2];
  int32_t parent[kMaxAlpha * 2];
};

__device__ void make_code_lengths(uint8_t *len, const uint32_t *freq, int alpha, int max_len, HuffWork &W) {
  int32_t *heap = W.heap, *weight = W.weight, *parent = W.parent;
  for (int i = 0; i < alpha; ++i) weight[i + 1] = (int32_t)((freq[i] == 0 ? 1u : freq[i]) << 8);
  for (;;) {
    int n_nodes = alpha, n_heap = 0;
    heap[0] = 0;
    weight[0] = 0;
    parent[0] = -2;
    auto upheap = [&](int z) {
      const int tmp = heap[z];
      while (weight[tmp] < weight[heap[z >> 1]]) {
        heap[z] = heap[z >> 1];
        z >>= 1;
      }
      heap[z] = tmp;
    };
    auto downheap = [&](int z) {
      const int tmp = heap[z];
      for (;;) {
        int y = z << 1;
        if (y > n_heap) break;
        if (y < n_heap && weight[heap[y + 1]] < weight[heap[y]]) y++;
        if (weight[tmp] < weight[heap[y]]) break;
        heap[z] = heap[y];
        z = y;
      }
      heap[z] = tmp;
    };
    for (int i = 1; i <= alpha; ++i) {
      parent[i] = -1;
      heap[++n_heap] = i;
      upheap(n_heap);
    }
    while (n_heap > 1) {
      const int n1 = heap[1];
      heap[1] = heap[n_heap--];
      downheap(1);
      const int n2 = heap[1];
      heap[1] = heap[n_heap--];
      downheap(1);
      ++n_nodes;
      parent[n1] = parent[n2] = n_nodes;
      const int32_t w1 = weight[n1], w2 = weight[n2];
      const int32_t d1 = w1 & 0xFF, d2 = w2 & 0xFF;
      weight[n_nodes] = (int32_t)(((uint32_t)w1 & 0xFFFFFF00u) + ((uint32_t)w2 & 0xFFFFFF00u)) |
                        (1 + (d1 > d2 ? d1 : d2));
      parent[n_nodes] = -1;
      heap[++n_heap] = n_nodes;
      upheap(n_heap);
    }
    bool too_long = false;
    for (int i = 1; i <= alpha; ++i) {
      int j = 0, k = i;
      while (parent[k] >= 0) {
        k = parent[k];
        ++j;
      }
      len[i - 1] = (uint8_t)j;
      too_long |= j > max_len;
    }
    if (!too_long) return;
    for (int i = 1; i <= alpha; ++i) {
      const int j = weight[i] >> 8;
      weight[i] = (1 + j / 2) << 8;
    }
  }
}

struct TablesOut {
  uint8_t len[kMaxGroups][kMaxAlpha];
  uint32_t code[kMaxGroups][kMaxAlpha];
};

__global__ void __launch_bounds__(kTableThreads) tables_kernel(Block *blocks, const int *ids,
                                                               const uint16_t *mtfv,
                                                               const uint32_t *freq_in,
                                                               uint8_t *selectors, uint8_t *sel_mtf,
                                                               TablesOut *tables) {
  Block &B = blocks[ids[blockIdx.x]];
  if (B.tie) return;
  __shared__ uint8_t len[kMaxGroups][kMaxAlpha];
  __shared__ uint32_t rfreq[kMaxGroups][kMaxAlpha];
  __shared__ uint32_t freq[kMaxAlpha];
  __shared__ unsigned long long data_bits;
  __shared__ HuffWork hw[kMaxGroups];
  __shared__ int32_t chunk_last[kTableThreads][kMaxGroups];
  __shared__ unsigned long long sel_bits_sum;
  const int tid = threadIdx.x;
  const int alpha = B.n_in_use + 2;
  const int n_mtf = B.n_mtf;
  const int n_groups = n_mtf < 200 ? 2 : n_mtf < 600 ? 3 : n_mtf < 1200 ? 4 : n_mtf < 2400 ? 5 : 6;
  const int n_sel = (n_mtf + kGroupSize - 1) / kGroupSize;
  const uint16_t *mv = mtfv + B.mtf_off;
  uint8_t *sel = selectors + B.sel_off;
  for (int i = tid; i < kMaxAlpha; i += blockDim.x) freq[i] = freq_in[(size_t)ids[blockIdx.x] * kMaxAlpha + i];
  __syncthreads();
  if (tid == 0) {  // initial partition of the symbol range into n_groups tables
    int n_part = n_groups, rem_f = n_mtf, gs = 0;
    while (n_part > 0) {
      const int t_freq = rem_f / n_part;
      int ge = gs - 1, a_freq = 0;
      while (a_freq < t_freq && ge < alpha - 1) a_freq += (int)freq[++ge];
      if (ge > gs && n_part != n_groups && n_part != 1 && ((n_groups - n_part) % 2 == 1))
        a_freq -= (int)freq[ge--];
      for (int v = 0; v < alpha; ++v) len[n_part - 1][v] = (v >= gs && v <= ge) ? 0 : 15;
      n_part--;
      gs = ge + 1;
      rem_f -= a_freq;
    }
  }
  __syncthreads();
  for (int iter = 0; iter < 4; ++iter) {
    for (int i = tid; i < kMaxGroups * kMaxAlpha; i += blockDim.x) (&rfreq[0][0])[i] = 0;
    __syncthreads();
    for (int g = tid; g < n_sel; g += blockDim.x) {
      const int gs = g * kGroupSize, ge = min(gs + kGroupSize, n_mtf);
      uint32_t cost[kMaxGroups] = {0, 0, 0, 0, 0, 0};
      for (int i = gs; i < ge; ++i) {
        const int v = mv[i];
#pragma unroll
        for (int t = 0; t < kMaxGroups; ++t)
          if (t < n_groups) cost[t] += len[t][v];
      }
      int bt = 0;
      uint32_t bc = cost[0];
      for (int t = 1; t < n_groups; ++t)
        if (cost[t] < bc) { bc = cost[t]; bt = t; }
      sel[g] = (uint8_t)bt;
      for (int i = gs; i < ge; ++i) atomicAdd(&rfreq[bt][mv[i]], 1u);
    }
    __syncthreads();
    // one table per warp (lane 0): the heap builds run on different schedulers
    if ((tid & 31) == 0 && (tid >> 5) < n_groups)
      make_code_lengths(len[tid >> 5], rfreq[tid >> 5], alpha, kMaxCodeLen, hw[tid >> 5]);
    __syncthreads();
  }
  TablesOut &T = tables[ids[blockIdx.x]];
  if (tid < n_groups) {  // BZ2_hbAssignCodes
    int mn = 32, mx = 0;
    for (int i = 0; i < alpha; ++i) {
      mn = min(mn, (int)len[tid][i]);
      mx = max(mx, (int)len[tid][i]);
    }
    uint32_t vec = 0;
    for (int n = mn; n <= mx; ++n) {
      for (int i = 0; i < alpha; ++i)
        if (len[tid][i] == n) T.code[tid][i] = vec++;
      vec <<= 1;
    }
    for (int i = 0; i < alpha; ++i) T.len[tid][i] = len[tid][i];
  }
  if (tid == 0) data_bits = 0;
  __syncthreads();
  unsigned long long mine = 0;
  for (int i = tid; i < n_mtf; i += blockDim.x) mine += len[sel[i / kGroupSize]][mv[i]];
  atomicAdd(&data_bits, mine);
  // selector MTF (compress.c sendMTFValues) in parallel: the MTF index of
  // selector i is the number of other tables whose latest use before i is
  // more recent than that of sel[i] (the initial list order 0, 1, ... acts
  // as uses at times -1, -2, ...).  Each thread owns a contiguous run of
  // selectors; the latest use per table before each run comes from a scan
  // of the per-run latest uses.
  {
    const int per = (n_sel + kTableThreads - 1) / kTableThreads;
    const int a = min(n_sel, tid * per), b = min(n_sel, a + per);
    int32_t last[kMaxGroups];
    for (int t = 0; t < kMaxGroups; ++t) last[t] = -1 - t;
    for (int i = a; i < b; ++i) last[sel[i]] = i;
    for (int t = 0; t < kMaxGroups; ++t) chunk_last[tid][t] = last[t];
    if (tid == 0) sel_bits_sum = 0;
    __syncthreads();
    if (tid < kMaxGroups) {   // exclusive running max over the runs, per table
      int32_t run = -1 - tid;
      for (int k = 0; k < kTableThreads; ++k) {
        const int32_t v = chunk_last[k][tid];
        chunk_last[k][tid] = run;
        run = max(run, v);
      }
    }
    __syncthreads();
    for (int t = 0; t < kMaxGroups; ++t) last[t] = chunk_last[tid][t];
    uint8_t *sm = sel_mtf + B.sel_off;
    unsigned long long bits = 0;
    for (int i = a; i < b; ++i) {
      const int s0 = sel[i];
      int j = 0;
      for (int t = 0; t < n_groups; ++t) j += (t != s0 && last[t] > last[s0]) ? 1 : 0;
      sm[i] = (uint8_t)j;
      bits += (unsigned long long)(j + 1);
      last[s0] = i;
    }
    atomicAdd(&sel_bits_sum, bits);
    __syncthreads();
  }
  if (tid == 0) {
    const int64_t sel_bits = (int64_t)sel_bits_sum;
    int used16 = 0;
    for (int i = 0; i < 16; ++i) used16 += ((B.in_use[i >> 1] >> ((i & 1) * 16)) & 0xFFFFu) ? 1 : 0;
    int64_t tab_bits = 0;
    for (int t = 0; t < n_groups; ++t) {
      int curr = len[t][0];
      tab_bits += 5;
      for (int i = 0; i < alpha; ++i) {
        const int l = len[t][i];
        tab_bits += 2 * (int64_t)abs(l - curr) + 1;
        curr = l;
      }
    }
    B.n_groups = n_groups;
    B.n_sel = n_sel;
    B.hdr_bits = 48 + 32 + 1 + 24 + 16 + 16 * used16 + 3 + 15 + sel_bits + tab_bits;
  }
  __syncthreads();
  if (tid == 0) B.data_bits = (int64_t)data_bits;
}

// ---------------------------------------------------------------------------
// E: bit emission (big-endian bit order of bzlib.c bsW)
// ---------------------------------------------------------------------------

__device__ __forceinline__ void put_bits(uint32_t *w, uint64_t bit, uint32_t v, int n) {
  if (n == 0) return;
  const uint64_t wi = bit >> 5;
  const int off = (int)(bit & 31);
  if (off + n <= 32) {
    atomicOr(w + wi, v << (32 - off - n));
  } else {
    const int hi = 32 - off, lo = n - hi;
    atomicOr(w + wi, v >> lo);
    atomicOr(w + wi + 1, v << (32 - lo));
  }
}

__global__ void __launch_bounds__(kEmitThreads) emit_kernel(const Block *blocks, const int *ids,
                                                             const uint16_t *mtfv,
                                                             const uint8_t *selectors,
                                                             const uint8_t *sel_mtf,
                                                             const TablesOut *tables, uint32_t *out) {
  const Block &B = blocks[ids[blockIdx.x]];
  if (B.tie) return;
  const TablesOut &T = tables[ids[blockIdx.x]];
  const int tid = threadIdx.x;
  const int alpha = B.n_in_use + 2;
  if (tid == 0) {
    uint64_t p = B.bit_off;
    auto put = [&](int n, uint32_t v) { put_bits(out, p, v, n); p += n; };
    put(24, 0x314159u);
    put(24, 0x265359u);
    put(32, B.crc);
    put(1, 0);
    put(24, (uint32_t)B.orig);
    uint32_t used16 = 0;
    for (int i = 0; i < 16; ++i)
      if ((B.in_use[i >> 1] >> ((i & 1) * 16)) & 0xFFFFu) used16 |= 1u << (15 - i);
    put(16, used16);
    for (int i = 0; i < 16; ++i) {
      const uint32_t h = (B.in_use[i >> 1] >> ((i & 1) * 16)) & 0xFFFFu;
      if (h) put(16, __brev(h) >> 16);  // bit for symbol 16i+j first
    }
    put(3, (uint32_t)B.n_groups);
    put(15, (uint32_t)B.n_sel);
    const uint8_t *sm = sel_mtf + B.sel_off;
    for (int i = 0; i < B.n_sel; ++i) {
      int j = sm[i] + 1;  // j ones then a zero
      while (j > 0) {
        const int k = j > 31 ? 31 : j;
        j -= k;
        put(k, j > 0 ? (1u << k) - 1u : ((1u << k) - 2u));
      }
    }
    for (int t = 0; t < B.n_groups; ++t) {
      int curr = T.len[t][0];
      put(5, (uint32_t)curr);
      for (int i = 0; i < alpha; ++i) {
        const int l = T.len[t][i];
        while (curr < l) { put(2, 2); ++curr; }
        while (curr > l) { put(2, 3); --curr; }
        put(1, 0);
      }
    }
  }
  // data: codes at scanned offsets
  typedef cub::BlockScan<unsigned long long, kEmitThreads> Scan;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ unsigned long long s_base;
  if (tid == 0) s_base = (unsigned long long)(B.bit_off + B.hdr_bits);
  __syncthreads();
  const uint16_t *mv = mtfv + B.mtf_off;
  const uint8_t *sel = selectors + B.sel_off;
  const int n_mtf = B.n_mtf;
  for (int tile = 0; tile < n_mtf; tile += kEmitThreads * kEmitItems) {
    const int i0 = tile + tid * kEmitItems;
    uint8_t l[kEmitItems];
    uint32_t c[kEmitItems];
    unsigned long long sum = 0;
#pragma unroll
    for (int q = 0; q < kEmitItems; ++q) {
      const int i = i0 + q;
      if (i < n_mtf) {
        const int t = sel[i / kGroupSize];
        const int v = mv[i];
        l[q] = T.len[t][v];
        c[q] = T.code[t][v];
      } else {
        l[q] = 0;
        c[q] = 0;
      }
      sum += l[q];
    }
    unsigned long long excl, total;
    Scan(scan_tmp).ExclusiveSum(sum, excl, total);
    uint64_t p = s_base + excl;
#pragma unroll
    for (int q = 0; q < kEmitItems; ++q) {
      put_bits(out, p, c[q], l[q]);
      p += l[q];
    }
    __syncthreads();
    if (tid == 0) s_base += total;
    __syncthreads();
  }
}

struct JobFrame {
  uint64_t bit0;      // absolute bit position of the job's stream
  uint64_t end_bit;   // position of the end-of-stream marker
  uint32_t combined;
};

__global__ void frame_kernel(const JobFrame *frames, const int *jids, int n, uint32_t *out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const JobFrame &F = frames[jids[t]];
  put_bits(out, F.bit0, 0x425A6839u, 32);  // "BZh9"
  put_bits(out, F.end_bit, 0x177245u, 24);
  put_bits(out, F.end_bit + 24, 0x385090u, 24);
  put_bits(out, F.end_bit + 48, F.combined, 32);
}

__global__ void byteswap_kernel(uint32_t *w, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    w[i] = __byte_perm(w[i], 0, 0x0123);
}

// ---------------------------------------------------------------------------
// host orchestration
// ---------------------------------------------------------------------------

thread_local std::string g_bz_err;

int bz_fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_bz_err = buf;
  return code;
}

#define BZ_TRY(x)                                                                             \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess)                                                                    \
      return bz_fail(PCBZ_E_CUDA, "%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, \
                     __LINE__);                                                               \
  } while (0)

struct Scratch {  // grow-only device buffers, one set per host thread
  struct Buf {
    void *p = nullptr;
    size_t cap = 0;
  };
  Buf b[48];
  template <typename T>
  int get(int slot, size_t count, T **out) {
    Buf &x = b[slot];
    const size_t need = std::max<size_t>(count * sizeof(T), 256);
    if (need > x.cap) {
      if (x.p) cudaFree(x.p);
      x.p = nullptr;
      x.cap = 0;
      BZ_TRY(cudaMalloc(&x.p, need));
      x.cap = need;
    }
    *out = static_cast<T *>(x.p);
    return PCBZ_OK;
  }
};
thread_local Scratch g_scr;

int grid_of(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 32));
}

__global__ void iota_kernel(uint32_t *a, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}

// Rotation sort of every block (stage B): sa[base + j] = start of the j-th
// smallest rotation of the block; blocks[b].tie set for periodic blocks.
int sort_rotations(Block *d_blocks, const int *d_ids, int nb, int nslots, const uint8_t *d_rle,
                   uint32_t N, uint32_t *sa, const std::vector<Block> &blocks, const std::vector<int> &ids,
                   cudaStream_t st) {
  uint32_t *block_of, *rank, *vals_a, *vals_b, *U, *U2, *gs;
  uint64_t *keys_a, *keys_b;
  uint8_t *hd, *unres;
  int *d_nsel;
  int rc;
  if ((rc = g_scr.get(4, N, &block_of)) || (rc = g_scr.get(6, N, &rank)) || (rc = g_scr.get(7, N, &vals_a)) ||
      (rc = g_scr.get(8, N, &vals_b)) || (rc = g_scr.get(9, N, &U)) || (rc = g_scr.get(10, N, &U2)) ||
      (rc = g_scr.get(11, N, &gs)) || (rc = g_scr.get(12, N, &keys_a)) || (rc = g_scr.get(13, N, &keys_b)) ||
      (rc = g_scr.get(14, N, &hd)) || (rc = g_scr.get(15, N, &unres)) || (rc = g_scr.get(16, 1, &d_nsel)))
    return rc;
  uint32_t *rs_totals, *rs_ctr;
  unsigned long long *rs_status, *rs_mask;
  uint32_t *rs_tables;
  if ((rc = g_scr.get(39, (size_t)256 * (rsort::tiles_of(N) + nb + 1), &rs_status)) ||
      (rc = g_scr.get(40, (size_t)8 * 256 * std::max(nb, 1), &rs_totals)) || (rc = g_scr.get(41, 1, &rs_mask)) ||
      (rc = g_scr.get(42, 8, &rs_ctr)) ||
      (rc = g_scr.get(43, (size_t)4 * nb + rsort::tiles_of(N) + nb + 2, &rs_tables)))
    return rc;
  uint64_t *ks;   // the sorted pairs: keys_b / vals_b or keys_a / vals_a
  uint32_t *vs;
  size_t t_scan = 0, t_sel = 0;
  BZ_TRY(cub::DeviceScan::InclusiveScan(nullptr, t_scan, gs, gs, MaxOp(), N, st));
  BZ_TRY(cub::DeviceSelect::Flagged(nullptr, t_sel, U, unres, U2, d_nsel, N, st));
  const size_t t_all = std::max(t_scan, t_sel);
  uint8_t *d_tmp;
  if ((rc = g_scr.get(17, t_all, &d_tmp))) return rc;
  int bits_b = 1;
  while ((1 << bits_b) < nslots) ++bits_b;
  int bits_r = 1;
  while (((uint64_t)1 << bits_r) <= (uint64_t)N) ++bits_r;
  fill_block_of_kernel<<<nb, 256, 0, st>>>(d_blocks, d_ids, block_of);
  init_keys_kernel<<<grid_of(N), 256, 0, st>>>(d_blocks, block_of, d_rle, N, keys_a, vals_a);
  BZ_TRY(cudaGetLastError());
  size_t tb = t_all;
  // first sort: the pairs already lie in their blocks' ranges in block order,
  // so each block's range is sorted by its 4-byte prefixes alone (segmented;
  // the block-id passes of a global sort by (block, prefix) are not needed)
  static const bool seg_first = getenv("PCBZ_RSORT_SEG") ? atoi(getenv("PCBZ_RSORT_SEG")) != 0 : true;
  if (seg_first) {
    std::vector<uint32_t> seg_base(nb), seg_n(nb);
    for (int t = 0; t < nb; ++t) {
      seg_base[t] = (uint32_t)blocks[ids[t]].base;
      seg_n[t] = (uint32_t)blocks[ids[t]].n;
    }
    BZ_TRY(rsort::sort_pairs_segmented(keys_a, vals_a, keys_b, vals_b, N, 32, seg_base, seg_n, rs_tables, rs_status,
                                       rs_totals, rs_ctr, rs_mask, &ks, &vs, st));
  } else {
    BZ_TRY(rsort::sort_pairs(keys_a, vals_a, keys_b, vals_b, N, 32 + bits_b, rs_status, rs_totals, rs_ctr, rs_mask,
                             &ks, &vs, st));
  }
  heads_kernel<<<grid_of(N), 256, 0, st>>>(ks, N, hd);
  head_pos_kernel<<<grid_of(N), 256, 0, st>>>(hd, nullptr, N, gs);
  tb = t_all;
  BZ_TRY(cub::DeviceScan::InclusiveScan(d_tmp, tb, gs, gs, MaxOp(), N, st));
  settle_kernel<<<grid_of(N), 256, 0, st>>>(vs, nullptr, N, hd, gs, sa, rank, block_of, d_blocks, 4, unres);
  uint32_t *idx = vs == vals_a ? vals_b : vals_a;   // the value buffer settle_kernel does not read
  iota_kernel<<<grid_of(N), 256, 0, st>>>(idx, N);
  tb = t_all;
  BZ_TRY(cub::DeviceSelect::Flagged(d_tmp, tb, idx, unres, U, d_nsel, N, st));
  int h_nsel = 0;
  BZ_TRY(cudaMemcpyAsync(&h_nsel, d_nsel, sizeof(int), cudaMemcpyDeviceToHost, st));
  BZ_TRY(cudaStreamSynchronize(st));
  uint32_t m = (uint32_t)h_nsel;
  static const bool trace = getenv("PCBZ_HOST_TRACE") != nullptr;
  if (trace) fprintf(stderr, "bwt: N %u, unresolved after 4-byte keys %u\n", N, m);
  for (uint64_t h = 4; m > 0; h *= 2) {
    pair_keys_kernel<<<grid_of(m), 256, 0, st>>>(U, m, sa, rank, block_of, d_blocks, h, keys_a, vals_a);
    tb = t_all;
    BZ_TRY(rsort::sort_pairs(keys_a, vals_a, keys_b, vals_b, m, 32 + bits_r, rs_status, rs_totals, rs_ctr, rs_mask, &ks, &vs, st));
    heads_kernel<<<grid_of(m), 256, 0, st>>>(ks, m, hd);
    head_pos_kernel<<<grid_of(m), 256, 0, st>>>(hd, U, m, gs);
    tb = t_all;
    BZ_TRY(cub::DeviceScan::InclusiveScan(d_tmp, tb, gs, gs, MaxOp(), m, st));
    settle_kernel<<<grid_of(m), 256, 0, st>>>(vs, U, m, hd, gs, sa, rank, block_of, d_blocks, 2 * h, unres);
    tb = t_all;
    BZ_TRY(cub::DeviceSelect::Flagged(d_tmp, tb, U, unres, U2, d_nsel, m, st));
    BZ_TRY(cudaMemcpyAsync(&h_nsel, d_nsel, sizeof(int), cudaMemcpyDeviceToHost, st));
    BZ_TRY(cudaStreamSynchronize(st));
    m = (uint32_t)h_nsel;
    if (trace) fprintf(stderr, "bwt: unresolved after %llu-byte prefixes %u\n", (unsigned long long)(2 * h), m);
    std::swap(U, U2);
  }
  return PCBZ_OK;
}

// c_zero_shift[k] = matrix of "append 2^k zero bytes" to the CRC register
int upload_zero_shift(cudaStream_t st) {
  static bool done = false;
  if (done) return PCBZ_OK;
  uint32_t tab[256];
  for (uint32_t i = 0; i < 256; ++i) {
    uint32_t c = i << 24;
    for (int k = 0; k < 8; ++k) c = (c & 0x80000000u) ? (c << 1) ^ 0x04C11DB7u : (c << 1);
    tab[i] = c;
  }
  static uint32_t P[32][32];
  for (int b = 0; b < 32; ++b) {
    const uint32_t v = 1u << b;
    P[0][b] = (v << 8) ^ tab[v >> 24];
  }
  auto apply = [](const uint32_t *M, uint32_t v) {
    uint32_t r = 0;
    for (int b = 0; b < 32; ++b)
      if (v & (1u << b)) r ^= M[b];
    return r;
  };
  for (int k = 1; k < 32; ++k)
    for (int b = 0; b < 32; ++b) P[k][b] = apply(P[k - 1], apply(P[k - 1], 1u << b));
  BZ_TRY(cudaMemcpyToSymbolAsync(c_zero_shift, P, sizeof P, 0, cudaMemcpyHostToDevice, st));
  BZ_TRY(cudaStreamSynchronize(st));
  done = true;
  return PCBZ_OK;
}

size_t job_bound(int64_t len) { return (size_t)((len + len / 100 + 1024 + 3) & ~(int64_t)3); }

const char *last_error() { return g_bz_err.c_str(); }

// Code jobs held in device memory (in_off: host array of njobs + 1 offsets
// into d_in).  Job j's bytes land at d_out + out_start[j] (4-byte aligned),
// out_len[j] bytes; host_needed[j] = 1 marks a job left to the host libbz2
// (a periodic block), with out_len[j] = 0.  Synchronises `st`.
int compress_jobs(const uint8_t *d_in, const int64_t *in_off, int njobs, uint8_t *d_out, size_t out_cap,
                  int64_t *out_start, int64_t *out_len, uint8_t *host_needed, cudaStream_t st) {
  if (njobs <= 0) return PCBZ_OK;
  for (int j = 0; j < njobs; ++j)
    if (in_off[j + 1] < in_off[j]) return bz_fail(PCBZ_E_INVALID, "job offsets must be non-decreasing");
  if (int rc0 = upload_zero_shift(st)) return rc0;
  // ---- A: RLE1 + block split ---------------------------------------------------
  const int64_t base_off = in_off[0];
  const int64_t total = in_off[njobs] - base_off;
  if (total >= ((int64_t)1 << 31)) return bz_fail(PCBZ_E_INVALID, "bzip2 batch too large: split the jobs");
  d_in += base_off;
  std::vector<int64_t> rel(njobs + 1);
  for (int j = 0; j <= njobs; ++j) rel[j] = in_off[j] - base_off;
  std::vector<Job> jobs(njobs);
  int nslots = 0;
  for (int j = 0; j < njobs; ++j) {
    Job &J = jobs[j];
    J.in_off = rel[j];
    J.in_len = rel[j + 1] - rel[j];
    J.rle_off = 0;
    J.block0 = nslots;
    nslots += (int)((J.in_len + J.in_len / 4 + 64) / kBlockMax) + 2;
    J.nblocks = 0;
  }
  nslots = std::max(nslots, 1);
  Job *d_jobs;
  Block *d_blocks;
  uint8_t *d_rle, *d_flags;
  int64_t *d_rel;
  uint32_t *d_rs, *d_iota, *d_osz, *d_acc, *d_chunk0;
  int *d_cnt;
  int rc;
  const int64_t T = std::max<int64_t>(total, 1);
  if ((rc = g_scr.get(0, njobs, &d_jobs)) || (rc = g_scr.get(1, nslots, &d_blocks)) ||
      (rc = g_scr.get(2, (size_t)(T + T / 4 + 64), &d_rle)) || (rc = g_scr.get(25, T, &d_flags)) ||
      (rc = g_scr.get(26, njobs + 1, &d_rel)) || (rc = g_scr.get(27, T + 1, &d_rs)) ||
      (rc = g_scr.get(28, T + 1, &d_iota)) || (rc = g_scr.get(29, T + 1, &d_osz)) ||
      (rc = g_scr.get(30, 1, &d_cnt)))
    return rc;
  BZ_TRY(cudaMemcpyAsync(d_jobs, jobs.data(), njobs * sizeof(Job), cudaMemcpyHostToDevice, st));
  BZ_TRY(cudaMemcpyAsync(d_rel, rel.data(), (njobs + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  uint32_t R = 0;
  if (total > 0) {
    run_flags_kernel<<<grid_of(total), 256, 0, st>>>(d_in, total, d_flags);
    job_start_flags_kernel<<<(njobs + 127) / 128, 128, 0, st>>>(d_rel, njobs, d_flags);
    iota64_kernel<<<grid_of(total), 256, 0, st>>>(d_iota, total);
    size_t tb = 0;
    BZ_TRY(cub::DeviceSelect::Flagged(nullptr, tb, d_iota, d_flags, d_rs, d_cnt, (int)total, st));
    uint8_t *d_tmp;
    if ((rc = g_scr.get(17, tb, &d_tmp))) return rc;
    BZ_TRY(cub::DeviceSelect::Flagged(d_tmp, tb, d_iota, d_flags, d_rs, d_cnt, (int)total, st));
    int h_cnt = 0;
    BZ_TRY(cudaMemcpyAsync(&h_cnt, d_cnt, sizeof(int), cudaMemcpyDeviceToHost, st));
    BZ_TRY(cudaStreamSynchronize(st));
    R = (uint32_t)h_cnt;
    run_sizes_kernel<<<grid_of(R), 256, 0, st>>>(d_rs, R, (uint32_t)total, d_osz);
    BZ_TRY(cudaMemsetAsync(d_osz + R, 0, sizeof(uint32_t), st));
    tb = 0;
    BZ_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, d_osz, d_iota, R + 1, st));
    if ((rc = g_scr.get(17, tb, &d_tmp))) return rc;
    BZ_TRY(cub::DeviceScan::ExclusiveSum(d_tmp, tb, d_osz, d_iota, R + 1, st));   // d_iota := ocum
    split_kernel<<<(njobs + 127) / 128, 128, 0, st>>>(d_rel, njobs, d_rs, R, (uint32_t)total, d_iota, d_jobs,
                                                      d_blocks);
    run_write_kernel<<<grid_of(R), 256, 0, st>>>(d_in, d_rs, R, (uint32_t)total, d_iota, d_rle);
    BZ_TRY(cudaGetLastError());
  }
  std::vector<Block> blocks(nslots);
  BZ_TRY(cudaMemcpyAsync(jobs.data(), d_jobs, njobs * sizeof(Job), cudaMemcpyDeviceToHost, st));
  BZ_TRY(cudaMemcpyAsync(blocks.data(), d_blocks, nslots * sizeof(Block), cudaMemcpyDeviceToHost, st));
  BZ_TRY(cudaStreamSynchronize(st));
  if (total == 0)
    for (int j = 0; j < njobs; ++j) jobs[j].nblocks = 0;
  std::vector<int> ids;
  int64_t N = 0, mtf_total = 0, sel_total = 0;
  for (int j = 0; j < njobs; ++j)
    for (int k = 0; k < jobs[j].nblocks; ++k) {
      const int b = jobs[j].block0 + k;
      Block &B = blocks[b];
      B.base = (uint32_t)N;
      B.mtf_off = mtf_total;
      B.sel_off = sel_total;
      N += B.n;
      mtf_total += B.n + 1;
      sel_total += (B.n + 1 + kGroupSize - 1) / kGroupSize;
      ids.push_back(b);
    }
  const int nb = (int)ids.size();
  if (N >= ((int64_t)1 << 31)) return bz_fail(PCBZ_E_INVALID, "bzip2 batch too large: split the jobs");
  int *d_ids;
  uint16_t *mtfv;
  uint32_t *freq, *sa;
  uint8_t *selectors, *sel_mtf;
  TablesOut *tables;
  if ((rc = g_scr.get(3, std::max(nb, 1), &d_ids)) || (rc = g_scr.get(5, std::max<int64_t>(N, 1), &sa)) ||
      (rc = g_scr.get(18, std::max<int64_t>(mtf_total, 1), &mtfv)) ||
      (rc = g_scr.get(19, (size_t)nslots * kMaxAlpha, &freq)) ||
      (rc = g_scr.get(20, std::max<int64_t>(sel_total, 1), &selectors)) ||
      (rc = g_scr.get(21, std::max<int64_t>(sel_total, 1), &sel_mtf)) ||
      (rc = g_scr.get(22, (size_t)nslots, &tables)))
    return rc;
  if (nb > 0) {
    BZ_TRY(cudaMemcpyAsync(d_ids, ids.data(), nb * sizeof(int), cudaMemcpyHostToDevice, st));
    BZ_TRY(cudaMemcpyAsync(d_blocks, blocks.data(), nslots * sizeof(Block), cudaMemcpyHostToDevice, st));
    // block CRCs (chunked) and used-symbol maps
    std::vector<uint32_t> chunk0(nb + 1, 0);
    for (int t = 0; t < nb; ++t) {
      const Block &B = blocks[ids[t]];
      chunk0[t + 1] = chunk0[t] + (B.in_end - B.in_begin + kCrcChunk - 1) / kCrcChunk;
    }
    if ((rc = g_scr.get(31, nb + 1, &d_chunk0)) || (rc = g_scr.get(32, nb, &d_acc))) return rc;
    BZ_TRY(cudaMemcpyAsync(d_chunk0, chunk0.data(), (nb + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    BZ_TRY(cudaMemsetAsync(d_acc, 0, nb * sizeof(uint32_t), st));
    crc_chunks_kernel<<<(chunk0[nb] + 127) / 128, 128, 0, st>>>(d_in, d_blocks, d_ids, d_chunk0, nb, d_acc);
    block_meta_kernel<<<nb, 256, 0, st>>>(d_rle, d_blocks, d_ids, d_acc);
    BZ_TRY(cudaGetLastError());
    // ---- B, C, D ---------------------------------------------------------------
    if ((rc = sort_rotations(d_blocks, d_ids, nb, nslots, d_rle, (uint32_t)N, sa, blocks, ids, st))) return rc;
    // ---- C: MTF + zero-run coding --------------------------------------------
    {
      std::vector<uint32_t> seg0(nb + 1, 0);
      for (int t = 0; t < nb; ++t) seg0[t + 1] = seg0[t] + (uint32_t)((blocks[ids[t]].n + kMtfSeg - 1) / kMtfSeg);
      const uint32_t nseg = seg0[nb];
      uint32_t *d_seg0, *P, *cnt, *block_of;
      uint8_t *symseq, *ranks;
      int32_t *lastpos;
      if ((rc = g_scr.get(33, nb + 1, &d_seg0)) || (rc = g_scr.get(34, N, &symseq)) ||
          (rc = g_scr.get(35, N, &ranks)) || (rc = g_scr.get(36, (size_t)nseg * 256, &lastpos)) ||
          (rc = g_scr.get(37, N, &P)) || (rc = g_scr.get(38, N + 1, &cnt)) || (rc = g_scr.get(4, N, &block_of)))
        return rc;
      BZ_TRY(cudaMemcpyAsync(d_seg0, seg0.data(), (nb + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
      const int gw = (int)((nseg + kMtfWarps - 1) / kMtfWarps);
      mtf_gather_kernel<<<gw, 32 * kMtfWarps, 0, st>>>(d_blocks, d_ids, nb, d_seg0, sa, d_rle, symseq, lastpos);
      mtf_prefix_kernel<<<nb, 256, 0, st>>>(d_seg0, lastpos);
      mtf_rank_kernel<<<gw, 32 * kMtfWarps, 0, st>>>(d_blocks, d_ids, nb, d_seg0, symseq, lastpos, ranks);
      nz_pos_kernel<<<grid_of(N), 256, 0, st>>>(ranks, (uint32_t)N, P);
      size_t tb = 0;
      uint8_t *d_tmp;
      BZ_TRY(cub::DeviceScan::InclusiveScan(nullptr, tb, P, P, MaxOp(), (uint32_t)N, st));
      if ((rc = g_scr.get(17, tb, &d_tmp))) return rc;
      BZ_TRY(cub::DeviceScan::InclusiveScan(d_tmp, tb, P, P, MaxOp(), (uint32_t)N, st));
      run_count_kernel<<<grid_of(N + 1), 256, 0, st>>>(ranks, P, block_of, d_blocks, (uint32_t)N, cnt);
      tb = 0;
      BZ_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, cnt, (uint32_t)N + 1, st));
      if ((rc = g_scr.get(17, tb, &d_tmp))) return rc;
      BZ_TRY(cub::DeviceScan::ExclusiveSum(d_tmp, tb, cnt, cnt, (uint32_t)N + 1, st));
      run_write_mtf_kernel<<<grid_of(N), 256, 0, st>>>(ranks, P, cnt, block_of, d_blocks, (uint32_t)N, mtfv);
      mtf_tail_freq_kernel<<<nb, 256, 0, st>>>(d_blocks, d_ids, P, cnt, mtfv, freq);
      BZ_TRY(cudaGetLastError());
    }
    tables_kernel<<<nb, kTableThreads, 0, st>>>(d_blocks, d_ids, mtfv, freq, selectors, sel_mtf, tables);
    BZ_TRY(cudaGetLastError());
    BZ_TRY(cudaMemcpyAsync(blocks.data(), d_blocks, nslots * sizeof(Block), cudaMemcpyDeviceToHost, st));
    BZ_TRY(cudaStreamSynchronize(st));
  }
  // ---- E: output layout, emission, framing --------------------------------------
  std::vector<JobFrame> frames(njobs);
  std::vector<int> coded;
  int64_t word = 0;
  for (int j = 0; j < njobs; ++j) {
    bool tie = false;
    for (int k = 0; k < jobs[j].nblocks; ++k) tie |= blocks[jobs[j].block0 + k].tie != 0;
    host_needed[j] = tie ? 1 : 0;
    out_start[j] = word * 4;
    out_len[j] = 0;
    if (tie) continue;
    const uint64_t bit0 = (uint64_t)word * 32;
    uint64_t p = bit0 + 32;
    uint32_t combined = 0;
    for (int k = 0; k < jobs[j].nblocks; ++k) {
      Block &B = blocks[jobs[j].block0 + k];
      B.bit_off = (int64_t)p;
      p += (uint64_t)(B.hdr_bits + B.data_bits);
      combined = ((combined << 1) | (combined >> 31)) ^ B.crc;
    }
    frames[j] = JobFrame{bit0, p, combined};
    const uint64_t end = p + 80;
    out_len[j] = (int64_t)((end - bit0 + 7) / 8);
    word += (int64_t)((end - bit0 + 31) / 32);
    coded.push_back(j);
  }
  if ((size_t)word * 4 > out_cap) return bz_fail(PCBZ_E_INVALID, "bzip2 output buffer too small");
  JobFrame *d_frames;
  int *d_coded;
  if ((rc = g_scr.get(23, njobs, &d_frames)) || (rc = g_scr.get(24, std::max<size_t>(coded.size(), 1), &d_coded)))
    return rc;
  BZ_TRY(cudaMemcpyAsync(d_frames, frames.data(), njobs * sizeof(JobFrame), cudaMemcpyHostToDevice, st));
  if (!coded.empty())
    BZ_TRY(cudaMemcpyAsync(d_coded, coded.data(), coded.size() * sizeof(int), cudaMemcpyHostToDevice, st));
  uint32_t *out_w = reinterpret_cast<uint32_t *>(d_out);
  if (word > 0) BZ_TRY(cudaMemsetAsync(out_w, 0, (size_t)word * 4, st));
  if (nb > 0) {
    BZ_TRY(cudaMemcpyAsync(d_blocks, blocks.data(), nslots * sizeof(Block), cudaMemcpyHostToDevice, st));
    emit_kernel<<<nb, kEmitThreads, 0, st>>>(d_blocks, d_ids, mtfv, selectors, sel_mtf, tables, out_w);
  }
  if (!coded.empty())
    frame_kernel<<<((int)coded.size() + 127) / 128, 128, 0, st>>>(d_frames, d_coded, (int)coded.size(), out_w);
  if (word > 0) byteswap_kernel<<<grid_of(word), 256, 0, st>>>(out_w, word);
  BZ_TRY(cudaGetLastError());
  BZ_TRY(cudaStreamSynchronize(st));
  return PCBZ_OK;
}

}  // namespace bz
}  // namespace pcbz

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------

namespace {
thread_local cudaStream_t g_bz_stream = nullptr;
struct HostBufs { pcbz::bz::Scratch::Buf in, out; };
thread_local HostBufs g_bz_host;
int grow(pcbz::bz::Scratch::Buf &b, size_t n) {
  if (n <= b.cap) return PCBZ_OK;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
  cudaError_t e = cudaMalloc(&b.p, std::max<size_t>(n, 256));
  if (e != cudaSuccess) return pcbz::bz::bz_fail(PCBZ_E_CUDA, "cudaMalloc: %s", cudaGetErrorString(e));
  b.cap = std::max<size_t>(n, 256);
  return PCBZ_OK;
}
}  // namespace

extern "C" {

const char *pcbz_bzip2_last_error(void) { return pcbz::bz::g_bz_err.c_str(); }

size_t pcbz_bzip2_bound(const int64_t *in_off, int njobs) {
  size_t b = 0;
  for (int j = 0; j < njobs; ++j) b += pcbz::bz::job_bound(in_off[j + 1] - in_off[j]);
  return b;
}

int pcbz_bzip2_device(const uint8_t *d_in, const int64_t *in_off, int njobs, uint8_t *d_out, size_t out_cap,
                      int64_t *out_start, int64_t *out_len, uint8_t *host_needed, void *stream) {
  return pcbz::bz::compress_jobs(d_in, in_off, njobs, d_out, out_cap, out_start, out_len, host_needed,
                                 static_cast<cudaStream_t>(stream));
}

int pcbz_bzip2_host(const uint8_t *in, const int64_t *in_off, int njobs, uint8_t *out, size_t out_cap,
                    int64_t *out_start, int64_t *out_len, uint8_t *host_needed) {
  if (njobs <= 0) return PCBZ_OK;
  if (!g_bz_stream) {
    cudaError_t e = cudaStreamCreateWithFlags(&g_bz_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return pcbz::bz::bz_fail(PCBZ_E_NODEVICE, "no CUDA device: %s", cudaGetErrorString(e));
  }
  const int64_t total = in_off[njobs] - in_off[0];
  int rc;
  const size_t bound = pcbz_bzip2_bound(in_off, njobs);
  if ((rc = grow(g_bz_host.in, (size_t)std::max<int64_t>(total, 1))) || (rc = grow(g_bz_host.out, bound)))
    return rc;
  std::vector<int64_t> rel(njobs + 1);
  for (int j = 0; j <= njobs; ++j) rel[j] = in_off[j] - in_off[0];
  cudaStream_t st = g_bz_stream;
  if (total > 0 &&
      cudaMemcpyAsync(g_bz_host.in.p, in + in_off[0], (size_t)total, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return pcbz::bz::bz_fail(PCBZ_E_CUDA, "H2D copy failed");
  rc = pcbz::bz::compress_jobs(static_cast<const uint8_t *>(g_bz_host.in.p), rel.data(), njobs,
                               static_cast<uint8_t *>(g_bz_host.out.p), bound, out_start, out_len,
                               host_needed, st);
  if (rc) return rc;
  int64_t used = 0;
  for (int j = 0; j < njobs; ++j) used = std::max(used, out_start[j] + out_len[j]);
  if ((size_t)used > out_cap) return pcbz::bz::bz_fail(PCBZ_E_INVALID, "output buffer too small");
  if (used > 0 && cudaMemcpy(out, g_bz_host.out.p, (size_t)used, cudaMemcpyDeviceToHost) != cudaSuccess)
    return pcbz::bz::bz_fail(PCBZ_E_CUDA, "D2H copy failed");
  return PCBZ_OK;
}

}  // extern "C"
