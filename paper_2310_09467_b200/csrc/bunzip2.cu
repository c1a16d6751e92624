// bunzip2.cu -- bzip2 (libbzip2 1.0.8 stream format) decoding on the GPU for
// decompress_stack: the reference decodes every PCBZ block with
// bz2.decompress on host threads (pkg/src/pcbz/blocks.py:84-92 via
// pipeline.py:121-139; decompress.c / bzlib.c of libbzip2 1.0.8).
//
// Many payloads (one bzip2 stream per PCBZ block, ~5 bzip2 blocks each) are
// decoded together:
//   1  scan_magic_kernel   every bit position of every payload is tested for
//                          the 48-bit block magic 0x314159265359 (blocks are
//                          not byte-aligned and their starts are only known
//                          after decoding the previous block)
//   2  decode_block_kernel one warp per candidate: block header, selector
//                          MTF, delta-coded code lengths, canonical Huffman
//                          decode through a 10-bit lookup table (all lanes in
//                          lockstep), RUNA/RUNB, inverse MTF with the list in
//                          registers (8 entries per lane) -> the BWT last
//                          column L, the bit where the block ends.  The host keeps the
//                          candidates that chain from bit 32 of each stream
//                          (a spurious magic inside coded data never chains)
//   3  inverse BWT         stable multisplit of positions by L[i] -> the T
//                          vector of decompress.c (tt[cftab[L[i]]++] = i), then list
//                          ranking of the chain p <- T[p] from T[origPtr]
//                          with rulers every 256 positions: rulers walk to the
//                          next ruler, one thread per block ranks the rulers,
//                          rulers write their segments
//   4  rle1_kernel         one warp per block: inverse RLE1 (runs of four
//                          + count byte, unRLE_obuf_to_output_FAST) as a scan
//                          of a 5-state automaton; output lengths, then the
//                          bytes; block CRCs over 4 KB chunks combined in
//                          GF(2) (crc_chunks_kernel)
// The host checks every block CRC and each stream's combined CRC and
// end-of-stream marker.  Anything this decoder does not take (randomised
// blocks, a stream that does not chain, a periodic block whose rotation cycle
// is shorter than the block, trailing data, a CRC mismatch) is reported so the
// caller decodes that payload with libbzip2, which also produces the
// reference's exception for corrupt data.
#include <algorithm>
#include <string>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <vector>

namespace pcbz {
namespace bzd {

constexpr int kMaxCand = 1 << 20;          // candidate slots per call
constexpr int kSlot = 900000;              // L bytes per candidate (level 9 max)
constexpr int kRuler = 256;                // list-ranking ruler spacing (64: 57 ms, 256: 41 ms, 1024: 61 ms on C2)
constexpr int kMaxGroups = 6;
constexpr int kMaxAlpha = 258;
constexpr int kMaxCodeLen = 23;

struct Cand {
  int32_t stream;
  int32_t level;       // blockSize100k of the stream
  int64_t bit;         // bit offset of the block magic in the stream
  // filled by decode_block_kernel
  int64_t end_bit;     // bit after the block's EOB symbol
  uint32_t crc;        // stored block CRC
  int32_t orig;        // origPtr
  int32_t n;           // BWT length
  int32_t status;      // 0 = decoded
};

__device__ __forceinline__ uint32_t crc_entry(uint32_t i) {
  uint32_t c = i << 24;
  for (int k = 0; k < 8; ++k) c = (c & 0x80000000u) ? (c << 1) ^ 0x04C11DB7u : (c << 1);
  return c;
}

// ---- 1: block magic candidates ------------------------------------------------

__global__ void scan_magic_kernel(const uint8_t *in, const int64_t *off, int nstreams, int64_t total,
                                  int64_t *cand_key, int *ncand) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < total;
       b += (int64_t)gridDim.x * blockDim.x) {
    // stream of this byte
    int lo = 0, hi = nstreams - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (off[mid] <= b) lo = mid; else hi = mid - 1;
    }
    const int64_t s0 = off[lo], s1 = off[lo + 1];
    uint64_t w = 0;
    for (int k = 0; k < 8; ++k) w = (w << 8) | (b + k < s1 ? in[b + k] : 0u);
    for (int sh = 0; sh < 8; ++sh) {
      if (b + (sh + 48 + 7) / 8 > s1) break;
      if (((w >> (16 - sh)) & 0xFFFFFFFFFFFFull) == 0x314159265359ull) {
        const int i = atomicAdd(ncand, 1);
        if (i < kMaxCand) cand_key[i] = ((int64_t)lo << 40) | ((b - s0) * 8 + sh);
      }
    }
  }
}

// ---- 2: one block: header, Huffman, RUNA/RUNB, inverse MTF ---------------------

struct BitReader {       // MSB-first bit reader; every lane of a warp runs it in lockstep
  const uint8_t *p;      // the payload; the device buffer is padded, so reads may run past len
  int64_t len, pos;      // bytes of the stream, next byte to load
  uint64_t buf;
  int nb;
  __device__ void init(const uint8_t *p_, int64_t len_, int64_t bit) {
    p = p_; len = len_; pos = bit >> 3; buf = 0; nb = 0;
    refill();
    refill();
    nb -= (int)(bit & 7);
  }
  // 32 bits, big-endian; not inlined, so the hot loop branches around it
  // (every ~4 symbols) instead of executing it predicated on every symbol
  __device__ __noinline__ void refill() {
    const uint32_t w = ((uint32_t)p[pos] << 24) | ((uint32_t)p[pos + 1] << 16) |
                       ((uint32_t)p[pos + 2] << 8) | (uint32_t)p[pos + 3];
    buf = (buf << 32) | w;
    pos += 4;
    nb += 32;
  }
  __device__ __forceinline__ uint32_t peek(int n) {   // n <= 32
    if (nb < n) refill();
    return (uint32_t)(buf >> (nb - n)) & (uint32_t)((1ull << n) - 1);
  }
  __device__ __forceinline__ uint32_t get(int n) {    // n <= 32
    if (n == 0) return 0;
    if (nb < n) refill();
    nb -= n;
    return (uint32_t)(buf >> nb) & (uint32_t)((1ull << n) - 1);
  }
  __device__ __forceinline__ void skip(int n) { nb -= n; }
  __device__ int64_t bitpos() const { return pos * 8 - nb; }
  __device__ bool over() const { return bitpos() > len * 8; }
};

// hbCreateDecodeTables (huffman.c)
__device__ void create_decode_tables(int32_t *limit, int32_t *base, int32_t *perm, const uint8_t *length,
                                     int minLen, int maxLen, int alphaSize) {
  int pp = 0;
  for (int i = minLen; i <= maxLen; i++)
    for (int j = 0; j < alphaSize; j++)
      if (length[j] == i) perm[pp++] = j;
  for (int i = 0; i < kMaxCodeLen; i++) base[i] = 0;
  for (int i = 0; i < alphaSize; i++) base[length[i] + 1]++;
  for (int i = 1; i < kMaxCodeLen; i++) base[i] += base[i - 1];
  for (int i = 0; i < kMaxCodeLen; i++) limit[i] = 0;
  int vec = 0;
  for (int i = minLen; i <= maxLen; i++) {
    vec += (base[i + 1] - base[i]);
    limit[i] = vec - 1;
    vec <<= 1;
  }
  for (int i = minLen + 1; i <= maxLen; i++) base[i] = ((limit[i - 1] + 1) << 1) - base[i];
}

constexpr int kLutBits = 10;

struct DecodeScratch {   // per decoding warp, in shared memory
  int32_t limit[kMaxGroups][kMaxCodeLen];
  int32_t base[kMaxGroups][kMaxCodeLen];
  int32_t perm[kMaxGroups][kMaxAlpha];
  int32_t minLen[kMaxGroups];
  uint16_t lut[kMaxGroups][1 << kLutBits];   // sym << 5 | len for codes of <= kLutBits bits, else 0
  uint8_t len[kMaxGroups][kMaxAlpha];
  uint8_t seq[256];
};

constexpr int kDecodeWarps = 8;
constexpr int kMaxSel = 18002;   // BZ_MAX_SELECTORS

// One warp per candidate block.  Header and Huffman decoding are run by all
// lanes in lockstep (uniform values, broadcast shared loads); the inverse MTF
// list lives in registers, eight entries per lane (entry 8l + j = byte j of
// lane l), and moving entry nn to the front is one funnel step per lane.
__global__ void __launch_bounds__(32 * kDecodeWarps) decode_block_kernel(
    const uint8_t *in, const int64_t *off, Cand *cand, int ncand, uint8_t *L, uint8_t *sel_scratch) {
  extern __shared__ uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * kDecodeWarps + warp;
  if (c >= ncand) return;
  DecodeScratch &S = reinterpret_cast<DecodeScratch *>(smem)[warp];
  uint8_t *selector = sel_scratch + (size_t)c * kMaxSel;   // selectors in global scratch (L1-cached reads)
  Cand &C = cand[c];
  const uint8_t *p = in + off[C.stream];
  const int64_t plen = off[C.stream + 1] - off[C.stream];
  BitReader br;
  br.init(p, plen, C.bit);
  if (lane == 0) C.status = 1;
  // header (decompress.c BZ_X_BLKHDR_1 .. BZ_X_CODING_3)
  const uint32_t m1 = br.get(24), m2 = br.get(24);
  if (m1 != 0x314159u || m2 != 0x265359u) return;
  const uint32_t crc = br.get(32);
  if (br.get(1)) { if (lane == 0) C.status = 2; return; }  // randomised block (bzip2 < 0.9.5)
  const int32_t orig = (int32_t)br.get(24);
  const int nblockMAX = 100000 * C.level;
  if (orig < 0 || orig > 10 + nblockMAX) return;
  const uint32_t in16 = br.get(16);
  int n_in_use = 0;
  for (int i = 0; i < 16; ++i)
    if (in16 & (0x8000u >> i)) {
      const uint32_t bits = br.get(16);
      for (int j = 0; j < 16; ++j)
        if (bits & (0x8000u >> j)) {
          if (lane == 0) S.seq[n_in_use] = (uint8_t)(i * 16 + j);
          n_in_use++;
        }
    }
  if (n_in_use == 0) return;
  const int alpha = n_in_use + 2;
  const int n_groups = (int)br.get(3);
  if (n_groups < 2 || n_groups > kMaxGroups) return;
  int n_sel = (int)br.get(15);
  if (n_sel < 1) return;
  {
    uint8_t pos[kMaxGroups];
    for (int i = 0; i < n_groups; ++i) pos[i] = (uint8_t)i;
    for (int i = 0; i < n_sel; ++i) {
      int j = 0;
      while (br.get(1)) {
        if (++j >= n_groups) return;
      }
      if (br.over()) return;
      if (i < kMaxSel) {
        const uint8_t tmp = pos[j];
        for (int v = j; v > 0; --v) pos[v] = pos[v - 1];
        pos[0] = tmp;
        if (lane == 0) selector[i] = tmp;
      }
    }
    if (n_sel > kMaxSel) n_sel = kMaxSel;
  }
  for (int t = 0; t < n_groups; ++t) {
    int curr = (int)br.get(5);
    for (int i = 0; i < alpha; ++i) {
      for (;;) {
        if (curr < 1 || curr > 20 || br.over()) return;
        if (!br.get(1)) break;
        if (!br.get(1)) curr++; else curr--;
      }
      if (lane == 0) S.len[t][i] = (uint8_t)curr;
    }
  }
  __syncwarp();
  for (int t = 0; t < n_groups; ++t) {
    int mn = 32, mx = 0;
    for (int i = 0; i < alpha; ++i) {
      mx = max(mx, (int)S.len[t][i]);
      mn = min(mn, (int)S.len[t][i]);
    }
    if (lane == 0) {
      create_decode_tables(S.limit[t], S.base[t], S.perm[t], S.len[t], mn, mx, alpha);
      S.minLen[t] = mn;
    }
    __syncwarp();
    // lookup table of the codes of <= kLutBits bits: the canonical decode of every prefix
    for (int e = lane; e < (1 << kLutBits); e += 32) {
      uint16_t ent = 0;
      for (int zn = mn; zn <= min(mx, kLutBits); ++zn) {
        const int32_t zvec = e >> (kLutBits - zn);
        if (zvec <= S.limit[t][zn]) {
          const int32_t k = zvec - S.base[t][zn];
          if (k >= 0 && k < kMaxAlpha) ent = (uint16_t)((S.perm[t][k] << 5) | zn);
          break;
        }
      }
      S.lut[t][e] = ent;
    }
  }
  __syncwarp();
  // MTF values
  uint64_t x = 0;
  for (int j = 0; j < 8; ++j) x |= (uint64_t)(8 * lane + j) << (8 * j);
  const int EOB = n_in_use + 1;
  int group_no = -1, group_pos = 0, gsel = 0;
  int32_t nblock = 0;
  uint8_t *o = L + (size_t)c * kSlot;   // next output byte (after the buffered ones)
  int pend = 0;                           // MTF bytes buffered in lanes 0..pend-1
  uint8_t obyte = 0;
  // Symbol decoding in two halves, so the lookup-table load of the next code
  // is in flight while the inverse MTF of the current symbol runs:
  // begin_sym (group bookkeeping, peek, LUT load) and end_sym (consume).
  auto begin_sym = [&](uint32_t &ent) -> bool {
    if (group_pos == 0) {
      if (++group_no >= n_sel) return false;
      group_pos = 50;
      gsel = selector[group_no];
    }
    group_pos--;
    ent = S.lut[gsel][br.peek(kLutBits)];
    return true;
  };
  auto end_sym = [&](uint32_t ent, int &sym) -> bool {
    if (ent & 31u) {
      br.skip((int)(ent & 31u));
      sym = (int)(ent >> 5);
      return true;
    }
    int zn = S.minLen[gsel];
    int32_t zvec = (int32_t)br.get(zn);
    for (;;) {
      if (zn > 20) return false;
      if (zvec <= S.limit[gsel][zn]) break;
      zn++;
      zvec = (zvec << 1) | (int32_t)br.get(1);
    }
    const int32_t k = zvec - S.base[gsel][zn];
    if (k < 0 || k >= kMaxAlpha) return false;
    sym = S.perm[gsel][k];
    return true;
  };
  auto next_sym = [&](int &sym) -> bool {
    uint32_t ent;
    return begin_sym(ent) && end_sym(ent, sym);
  };
  int sym;
  if (!next_sym(sym)) return;
  for (;;) {
    if (sym == EOB) break;
    if (sym <= 1) {  // RUNA / RUNB
      int32_t es = -1, N = 1;
      do {
        if (N >= 2 * 1024 * 1024) return;
        es += (sym + 1) * N;
        N *= 2;
        if (!next_sym(sym)) return;
      } while (sym <= 1);
      es++;
      const uint32_t front = (uint32_t)__shfl_sync(0xffffffffu, (uint32_t)x, 0) & 0xFFu;
      const uint8_t uc = S.seq[front];
      if (nblock + es > nblockMAX) return;
      if (pend) {            // the buffered MTF bytes precede the run
        if (lane < pend) o[lane] = obyte;
        o += pend;
        pend = 0;
      }
      for (int32_t k = lane; k < es; k += 32) o[k] = uc;
      nblock += es;
      o += es;
      continue;
    }
    if (nblock >= nblockMAX) return;
    // the next code's table entry is loaded first (its bits follow this
    // symbol's, which end_sym has already consumed)
    uint32_t ent;
    if (!begin_sym(ent)) return;
    // inverse MTF of index nn: entries 0..nn-1 move up one place, entry nn to the front
    const int nn = sym - 1;
    const int src = nn >> 3, b = nn & 7;
    const uint32_t v = __shfl_sync(0xffffffffu, (uint32_t)(x >> (8 * b)) & 0xFFu, src);
    const uint32_t top = __shfl_up_sync(0xffffffffu, (uint32_t)(x >> 56), 1);
    const uint64_t cin = lane == 0 ? v : top;
    // lanes below src shift all eight entries, lane src the ones below b
    const uint64_t lowmask = (1ull << (8 * b)) - 1;            // b <= 7
    const uint64_t keep = ~((lowmask << 8) | 0xFFull);         // entries above b
    const uint64_t shifted = (x << 8) | cin;
    const uint64_t partial = (x & keep) | ((x & lowmask) << 8) | cin;
    x = lane < src ? shifted : (lane == src ? partial : x);
    const uint8_t uc = S.seq[v];
    // lane `pend` keeps this byte; 32 of them leave as one coalesced store
    obyte = lane == pend ? uc : obyte;
    if (++pend == 32) {
      o[lane] = obyte;
      o += 32;
      pend = 0;
    }
    nblock++;
    if (!end_sym(ent, sym)) return;
  }
  if (pend && lane < pend) o[lane] = obyte;
  if (orig >= nblock || br.over()) return;
  if (lane == 0) {
    C.crc = crc;
    C.orig = orig;
    C.n = nblock;
    C.end_bit = br.bitpos();
    C.status = 0;
  }
}

// ---- 3: inverse BWT --------------------------------------------------------------

struct VBlock {          // a decoded block on a valid chain
  int32_t cand;          // its candidate slot (L bytes, counts)
  int32_t n, orig;
  int64_t base;          // first element in the concatenated element space
  int64_t r0;            // first ruler slot
  int32_t nr;            // ruler slots: ceil(n / kRuler) + 1 (the chain start)
  int32_t p0;            // chain start T[orig] (set on the device)
  int32_t status;
  int64_t out_off;       // RLE1 output offset (absolute)
  int64_t out_len;       // RLE1 output length (pass 1)
  uint32_t crc;          // computed block CRC (pass 2)
};

// T vector without a sort (decompress.c: tt[cftab[L[i]]++] = i): a stable
// multisplit of each block's positions by byte value over 4 KB chunks --
// per-chunk byte counts, per-block running offsets (one thread per byte
// value walks the chunks), then every chunk places its positions in order, a
// warp at a time, ranking equal bytes within the warp with __match_any_sync.
constexpr int kTChunk = 4096;

__global__ void tchunk_count_kernel(const VBlock *vb, const uint8_t *L, const int64_t *chunk_blk,
                                    const int32_t *chunk_idx, int64_t nchunks, uint32_t *counts) {
  __shared__ uint32_t h[256];
  const int64_t t = blockIdx.x;
  if (t >= nchunks) return;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const VBlock &B = vb[chunk_blk[t]];
  const uint8_t *Lb = L + (size_t)B.cand * kSlot;
  const int32_t a = chunk_idx[t] * kTChunk, e = min(B.n, a + kTChunk);
  for (int32_t i = a + threadIdx.x; i < e; i += blockDim.x) atomicAdd(&h[Lb[i]], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) counts[t * 256 + i] = h[i];
}

// one CTA of 256 threads per block: counts -> absolute starts of every (chunk, byte)
__global__ void __launch_bounds__(256) tchunk_offsets_kernel(const VBlock *vb, const int64_t *chunk0,
                                                             uint32_t *counts) {
  __shared__ uint32_t tot[256];
  const int b = blockIdx.x, c = threadIdx.x;
  const int64_t c0 = chunk0[b], c1 = chunk0[b + 1];
  uint32_t run = 0;
  for (int64_t t = c0; t < c1; ++t) {
    const uint32_t v = counts[t * 256 + c];
    counts[t * 256 + c] = run;
    run += v;
  }
  tot[c] = run;
  __syncthreads();
  uint32_t base = 0;   // cftab[c]: bytes below c in the block
  for (int k = 0; k < c; ++k) base += tot[k];
  for (int64_t t = c0; t < c1; ++t) counts[t * 256 + c] += base;
  (void)vb;
}

// one warp per chunk: T[start(byte) + rank] = position, in position order
__global__ void tchunk_place_kernel(const VBlock *vb, const uint8_t *L, const int64_t *chunk_blk,
                                    const int32_t *chunk_idx, int64_t nchunks, const uint32_t *starts,
                                    uint32_t *T) {
  __shared__ uint32_t next[4][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * 4 + warp;
  if (t >= nchunks) return;
  const VBlock &B = vb[chunk_blk[t]];
  const uint8_t *Lb = L + (size_t)B.cand * kSlot;
  uint32_t *Tb = T + B.base;
  uint32_t *nx = next[warp];
  for (int i = lane; i < 256; i += 32) nx[i] = starts[t * 256 + i];
  __syncwarp();
  const int32_t a = chunk_idx[t] * kTChunk, e = min(B.n, a + kTChunk);
  for (int32_t p0 = a; p0 < e; p0 += 32) {
    const int32_t p = p0 + lane;
    const bool valid = p < e;
    const uint32_t c = valid ? Lb[p] : 256u + lane;   // invalid lanes never match a byte
    const uint32_t peers = __match_any_sync(0xffffffffu, c);
    const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (valid && lane == leader) base = nx[c];
    base = __shfl_sync(0xffffffffu, base, leader);
    if (valid) Tb[base + rank] = (uint32_t)p;
    __syncwarp();
    if (valid && lane == leader) nx[c] = base + __popc(peers);
    __syncwarp();
  }
}

__device__ __forceinline__ bool is_ruler(int32_t q, int32_t p0) { return q % kRuler == 0 || q == p0; }
__device__ __forceinline__ int32_t ruler_slot(int32_t q, int32_t p0, int32_t nr) {
  return q % kRuler == 0 ? q / kRuler : nr - 1;
}

__global__ void chain_start_kernel(VBlock *vb, int nvb, const uint32_t *T) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nvb) vb[i].p0 = (int32_t)T[vb[i].base + vb[i].orig];
}

// every ruler walks to the next ruler: (next slot, segment length)
__global__ void ruler_walk_kernel(const VBlock *vb, int nvb, const uint32_t *T, const int64_t *ruler_blk,
                                  int64_t nrulers, int32_t *rnext, int32_t *rlen) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrulers;
       r += (int64_t)gridDim.x * blockDim.x) {
    const VBlock &B = vb[ruler_blk[r]];
    const int32_t k = (int32_t)(r - B.r0);
    int32_t p = k == B.nr - 1 ? B.p0 : k * kRuler;
    rlen[r] = -1;
    rnext[r] = -1;
    if (p >= B.n || (k == B.nr - 1 && B.p0 % kRuler == 0)) continue;   // empty slot
    const uint32_t *Tb = T + B.base;
    int32_t len = 1, q = (int32_t)Tb[p];
    while (!is_ruler(q, B.p0)) {
      q = (int32_t)Tb[q];
      if (++len > B.n) break;
    }
    rlen[r] = len;
    rnext[r] = ruler_slot(q, B.p0, B.nr);
  }
}

// one thread per block: ranks of the rulers along the chain from p0
__global__ void ruler_rank_kernel(VBlock *vb, int nvb, const int32_t *rnext, const int32_t *rlen,
                                  int32_t *rrank) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nvb) return;
  VBlock &B = vb[i];
  for (int32_t k = 0; k < B.nr; ++k) rrank[B.r0 + k] = -1;
  const int32_t start = ruler_slot(B.p0, B.p0, B.nr);
  int32_t s = start;
  int64_t rank = 0;
  for (;;) {
    if (rlen[B.r0 + s] < 0 || rrank[B.r0 + s] >= 0) { B.status = 3; return; }  // cycle shorter than n
    rrank[B.r0 + s] = (int32_t)rank;
    rank += rlen[B.r0 + s];
    if (rank >= B.n) break;
    s = rnext[B.r0 + s];
    if (s < 0 || s >= B.nr) { B.status = 3; return; }
  }
  if (rank != B.n) B.status = 3;
}

__global__ void ruler_write_kernel(const VBlock *vb, const uint32_t *T, const uint8_t *L,
                                   const int64_t *ruler_blk, int64_t nrulers, const int32_t *rlen,
                                   const int32_t *rrank, uint8_t *bwt_out) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrulers;
       r += (int64_t)gridDim.x * blockDim.x) {
    const VBlock &B = vb[ruler_blk[r]];
    if (B.status || rrank[r] < 0) continue;
    const int32_t k = (int32_t)(r - B.r0);
    int32_t q = k == B.nr - 1 ? B.p0 : k * kRuler;
    const uint32_t *Tb = T + B.base;
    const uint8_t *Lb = L + (size_t)B.cand * kSlot;
    uint8_t *o = bwt_out + B.base + rrank[r];
    const int32_t len = rlen[r];
    for (int32_t j = 0; j < len; ++j) {
      o[j] = Lb[q];
      q = (int32_t)Tb[q];
    }
  }
}

// ---- 4: inverse RLE1, then the block CRCs ------------------------------------------
//
// unRLE_obuf_to_output_FAST as a warp scan: the decoder is a 5-state
// automaton over the bytes -- A1..A4 (length of the current run of equal
// bytes) and C (a count byte was just consumed) -- whose transition depends
// only on whether a byte equals its predecessor:
//   equal:    A1->A2, A2->A3, A3->A4, A4->C, C->A1
//   unequal:  A1,A2,A3->A1, A4->C, C->A1
// A byte read in state A4 is a count: it stands for that many more copies of
// the previous byte.  32 bytes per step: transition maps composed by a warp
// scan (3 bits per state), copy counts prefix-summed, every lane writes its
// own bytes.

constexpr uint32_t kMapEq = 1u | 2u << 3 | 3u << 6 | 4u << 9 | 0u << 12;
constexpr uint32_t kMapNe = 0u | 0u << 3 | 0u << 6 | 4u << 9 | 0u << 12;
constexpr uint32_t kMapId = 0u | 1u << 3 | 2u << 6 | 3u << 9 | 4u << 12;

__device__ __forceinline__ uint32_t map_then(uint32_t f, uint32_t g) {   // g after f
  uint32_t r = 0;
#pragma unroll
  for (int st = 0; st < 5; ++st) r |= ((g >> (3 * ((f >> (3 * st)) & 7u))) & 7u) << (3 * st);
  return r;
}

// one warp per block: WRITE = false -> output lengths, true -> the bytes
template <bool WRITE>
__global__ void __launch_bounds__(128) rle1_kernel(VBlock *vb, int nvb, const uint8_t *bwt_out, uint8_t *out) {
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= nvb) return;
  VBlock &B = vb[i];
  if (B.status) return;
  const uint8_t *s = bwt_out + B.base;
  uint8_t *o = WRITE ? out + B.out_off : nullptr;
  const int32_t n = B.n;
  uint32_t state = 4;          // C: the first byte starts a run
  uint32_t pb = 0;
  int64_t olen = 0;
  for (int32_t base = 0; base < n; base += 32) {
    const int32_t j = base + lane;
    const bool valid = j < n;
    const uint32_t bj = valid ? s[j] : 0u;
    uint32_t prevb = __shfl_up_sync(0xffffffffu, bj, 1);
    if (lane == 0) prevb = pb;
    uint32_t f = valid ? (bj == prevb ? kMapEq : kMapNe) : kMapId;
    // inclusive scan: g = f_lane after ... after f_0
    uint32_t g = f;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t h = __shfl_up_sync(0xffffffffu, g, d);
      if (lane >= d) g = map_then(h, g);
    }
    uint32_t gx = __shfl_up_sync(0xffffffffu, g, 1);   // exclusive
    if (lane == 0) gx = kMapId;
    const uint32_t before = (gx >> (3 * state)) & 7u;
    const bool is_count = valid && before == 3;
    const uint32_t cnt = !valid ? 0u : (is_count ? bj : 1u);
    const uint8_t ch = (uint8_t)(is_count ? prevb : bj);
    uint32_t incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t h = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += h;
    }
    if (WRITE)
      for (uint32_t k = 0; k < cnt; ++k) o[olen + incl - cnt + k] = ch;
    olen += __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t gall = __shfl_sync(0xffffffffu, g, 31);
    state = (gall >> (3 * state)) & 7u;
    pb = __shfl_sync(0xffffffffu, bj, 31);
  }
  if (!WRITE && lane == 0) B.out_len = olen;
}

// Block CRCs (bzlib.c BZ_UPDATE_CRC, CRC-32/BZIP2) in parallel: each thread
// takes a 4 KB chunk of a block's output, computes its CRC from a zero
// register, shifts it over the bytes after the chunk (GF(2)-linear: powers of
// the "append one zero byte" matrix) and XORs it into the block's sum; the
// initial register's contribution is added once per block.
constexpr int kCrcChunk = 4096;

__global__ void crc_chunks_kernel(VBlock *vb, const int64_t *chunk_blk, const int32_t *chunk_idx,
                                  int64_t nchunks, const uint8_t *out, const uint32_t *zshift,
                                  uint32_t *crc_acc) {
  __shared__ uint32_t tab[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) tab[i] = crc_entry((uint32_t)i);
  __syncthreads();
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nchunks;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t bi = chunk_blk[t];
    const VBlock &B = vb[bi];
    const int64_t a = (int64_t)chunk_idx[t] * kCrcChunk;
    const int64_t e = a + kCrcChunk < B.out_len ? a + kCrcChunk : B.out_len;
    uint32_t c = 0;
    const uint8_t *p = out + B.out_off;
    for (int64_t k = a; k < e; ++k) c = (c << 8) ^ tab[(c >> 24) ^ p[k]];
    uint64_t after = (uint64_t)(B.out_len - e);
    for (int k = 0; after; ++k, after >>= 1)
      if (after & 1) {
        uint32_t r = 0;
        for (int bit = 0; bit < 32; ++bit)
          if (c & (1u << bit)) r ^= zshift[k * 32 + bit];
        c = r;
      }
    atomicXor(&crc_acc[bi], c);
  }
}

__global__ void crc_finish_kernel(VBlock *vb, int nvb, const uint32_t *zshift, const uint32_t *crc_acc) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nvb || vb[i].status) return;
  uint32_t c = 0xFFFFFFFFu;
  uint64_t n = (uint64_t)vb[i].out_len;
  for (int k = 0; n; ++k, n >>= 1)
    if (n & 1) {
      uint32_t r = 0;
      for (int bit = 0; bit < 32; ++bit)
        if (c & (1u << bit)) r ^= zshift[k * 32 + bit];
      c = r;
    }
  vb[i].crc = ~(c ^ crc_acc[i]);
}

}  // namespace bzd
}  // namespace pcbz

// ---- host orchestration -------------------------------------------------------------

namespace pcbz {
namespace bzd {

// big-endian residual stream (core.py:228-237) -> uint16 samples
__global__ void be16_kernel(const uint8_t *s, int64_t n, uint16_t *out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    out[k] = (uint16_t)((s[2 * k] << 8) | s[2 * k + 1]);
}

cudaError_t launch_be16(const uint8_t *s, int64_t n, uint16_t *out, cudaStream_t st) {
  be16_kernel<<<(int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 64)), 256, 0, st>>>(s, n, out);
  return cudaGetLastError();
}

namespace {

struct Buf {
  void *p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t n) {
    if (n <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    const size_t want = std::max<size_t>(n, 1 << 16);
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  template <typename T> T *as() const { return reinterpret_cast<T *>(p); }
};

struct Ctx {
  Buf in, off, ckey, ncand, cand, L, vb, vals2, rblk, rnext, rlen, rrank, bwt;
  Buf zs, crcacc, cblk, cidx, sel, tcb, tci, tc0, tcnt;
  bool zs_ready = false;
};
thread_local Ctx g;

#define BZD_TRY(x)                                                                  \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      err = std::string(#x) + ": " + cudaGetErrorString(e_);                        \
      return -2;                                                                    \
    }                                                                               \
  } while (0)

int grid_of(int64_t n, int t = 256) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + t - 1) / t, 65535 * 16)); }

uint64_t bits_at(const uint8_t *p, int64_t len, int64_t bit, int n) {  // n <= 56, MSB first
  uint64_t v = 0;
  for (int k = 0; k < n; ++k) {
    const int64_t b = bit + k;
    const int byte = (b >> 3) < len ? p[b >> 3] : 0;
    v = (v << 1) | ((byte >> (7 - (b & 7))) & 1);
  }
  return v;
}

// One batch of payloads (all with status still 1 on entry).
int decode_batch(const uint8_t *const *payloads, const int64_t *plen, const std::vector<int> &ids,
                 uint8_t *d_out, const int64_t *out_off, const int64_t *out_len, uint8_t *status,
                 cudaStream_t st, std::string &err) {
  static const bool trace = getenv("PCBZ_HOST_TRACE") != nullptr;
  using clk = std::chrono::steady_clock;
  auto t0 = clk::now();
  auto mark = [&](const char *what) {
    if (!trace) return;
    cudaStreamSynchronize(st);
    fprintf(stderr, "bunzip2 batch (%zu payloads): %s at %.2f ms\n", ids.size(), what,
            std::chrono::duration<double, std::milli>(clk::now() - t0).count());
  };
  const int ns = (int)ids.size();
  std::vector<int64_t> off(ns + 1, 0);
  std::vector<int> level(ns, 0);
  for (int s = 0; s < ns; ++s) {
    const uint8_t *p = payloads[ids[s]];
    const int64_t n = plen[ids[s]];
    if (n >= 14 && p[0] == 'B' && p[1] == 'Z' && p[2] == 'h' && p[3] >= '1' && p[3] <= '9') level[s] = p[3] - '0';
    off[s + 1] = off[s] + n;
  }
  const int64_t total = off[ns];
  if (total == 0) return 0;
  BZD_TRY(g.in.ensure((size_t)total + 64));   // padded: the bit reader loads 4 bytes at a time
  BZD_TRY(cudaMemsetAsync(g.in.as<uint8_t>() + total, 0, 64, st));
  BZD_TRY(g.off.ensure((size_t)(ns + 1) * 8));
  for (int s = 0; s < ns; ++s)
    if (plen[ids[s]]) BZD_TRY(cudaMemcpyAsync(g.in.as<uint8_t>() + off[s], payloads[ids[s]], (size_t)plen[ids[s]], cudaMemcpyHostToDevice, st));
  BZD_TRY(cudaMemcpyAsync(g.off.p, off.data(), (size_t)(ns + 1) * 8, cudaMemcpyHostToDevice, st));
  mark("upload");
  // 1: candidates
  BZD_TRY(g.ckey.ensure((size_t)kMaxCand * 8));
  BZD_TRY(g.ncand.ensure(4));
  BZD_TRY(cudaMemsetAsync(g.ncand.p, 0, 4, st));
  scan_magic_kernel<<<grid_of(total), 256, 0, st>>>(g.in.as<uint8_t>(), g.off.as<int64_t>(), ns, total,
                                                   g.ckey.as<int64_t>(), g.ncand.as<int>());
  int ncand = 0;
  BZD_TRY(cudaMemcpyAsync(&ncand, g.ncand.p, 4, cudaMemcpyDeviceToHost, st));
  BZD_TRY(cudaStreamSynchronize(st));
  // a real block holds >= ~700 KB of decoded bytes (RLE1 never expands a
  // 900 KB block below that) plus one partial block per stream: far more
  // magic candidates than that means adversarial data -- leave the batch to
  // libbzip2 rather than allocating a slot per candidate
  int64_t expect = 0;
  for (int s = 0; s < ns; ++s) expect += out_len[ids[s]] / 700000 + 1;
  if (ncand > kMaxCand || ncand > 4 * expect + 1024) return 0;
  std::vector<int64_t> key(ncand);
  if (ncand) BZD_TRY(cudaMemcpy(key.data(), g.ckey.p, (size_t)ncand * 8, cudaMemcpyDeviceToHost));
  std::sort(key.begin(), key.end());
  mark("magic scan");
  std::vector<Cand> cand(ncand);
  for (int i = 0; i < ncand; ++i) {
    memset(&cand[i], 0, sizeof(Cand));
    cand[i].stream = (int32_t)(key[i] >> 40);
    cand[i].bit = key[i] & ((1ll << 40) - 1);
    cand[i].level = std::max(1, level[cand[i].stream]);
    cand[i].status = 1;
  }
  // 2: decode every candidate
  if (ncand) {
    BZD_TRY(g.cand.ensure((size_t)ncand * sizeof(Cand)));
    BZD_TRY(g.L.ensure((size_t)ncand * kSlot));
    BZD_TRY(g.sel.ensure((size_t)ncand * kMaxSel));
    BZD_TRY(cudaMemcpyAsync(g.cand.p, cand.data(), (size_t)ncand * sizeof(Cand), cudaMemcpyHostToDevice, st));
    const size_t smem = kDecodeWarps * sizeof(DecodeScratch);
    BZD_TRY(cudaFuncSetAttribute(decode_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    decode_block_kernel<<<(ncand + kDecodeWarps - 1) / kDecodeWarps, 32 * kDecodeWarps, smem, st>>>(
        g.in.as<uint8_t>(), g.off.as<int64_t>(), g.cand.as<Cand>(), ncand, g.L.as<uint8_t>(), g.sel.as<uint8_t>());
    BZD_TRY(cudaMemcpyAsync(cand.data(), g.cand.p, (size_t)ncand * sizeof(Cand), cudaMemcpyDeviceToHost, st));
    BZD_TRY(cudaStreamSynchronize(st));
    mark("huffman + mtf decode");
  }
  // host: follow each stream's chain of blocks from bit 32 to the end-of-stream marker
  std::vector<VBlock> vb;
  std::vector<int> vb_stream;
  std::vector<uint32_t> vb_crc;
  std::vector<uint8_t> ok(ns, 0);
  std::vector<uint32_t> stored_comb(ns, 0);
  std::vector<std::pair<int, int>> range(ns, {0, 0});
  size_t ci = 0;
  for (int s = 0; s < ns; ++s) {
    while (ci < cand.size() && cand[ci].stream < s) ++ci;
    const size_t c0 = ci;
    size_t c1 = c0;
    while (c1 < cand.size() && cand[c1].stream == s) ++c1;
    if (!level[s]) continue;
    const uint8_t *p = payloads[ids[s]];
    const int64_t n = plen[ids[s]];
    int64_t bit = 32;
    const int vb0 = (int)vb.size();
    bool good = true;
    for (;;) {
      size_t c = c0;
      while (c < c1 && cand[c].bit < bit) ++c;
      if (c < c1 && cand[c].bit == bit) {
        if (cand[c].status != 0) { good = false; break; }
        VBlock B{};
        B.cand = (int32_t)c;
        B.n = cand[c].n;
        B.orig = cand[c].orig;
        vb.push_back(B);
        vb_stream.push_back(s);
        vb_crc.push_back(cand[c].crc);
        bit = cand[c].end_bit;
        continue;
      }
      // end of stream: marker, combined CRC, padding to the payload's end
      if (bits_at(p, n, bit, 48) != 0x177245385090ull || (bit + 80 + 7) / 8 != n) good = false;
      else stored_comb[s] = (uint32_t)bits_at(p, n, bit + 48, 32);
      break;
    }
    if (!good) {
      vb.resize(vb0);
      vb_stream.resize(vb0);
      vb_crc.resize(vb0);
      continue;
    }
    ok[s] = 1;
    range[s] = {vb0, (int)vb.size()};
  }
  const int nvb = (int)vb.size();
  if (nvb > (1 << 23)) return 0;
  int64_t tot = 0, nr = 0;
  std::vector<int64_t> rblk;
  for (int i = 0; i < nvb; ++i) {
    vb[i].base = tot;
    tot += vb[i].n;
    vb[i].nr = (vb[i].n + kRuler - 1) / kRuler + 1;
    vb[i].r0 = nr;
    nr += vb[i].nr;
  }
  if (nvb) {
    rblk.resize(nr);
    for (int i = 0; i < nvb; ++i)
      for (int k = 0; k < vb[i].nr; ++k) rblk[vb[i].r0 + k] = i;
    BZD_TRY(g.vb.ensure((size_t)nvb * sizeof(VBlock)));
    BZD_TRY(cudaMemcpyAsync(g.vb.p, vb.data(), (size_t)nvb * sizeof(VBlock), cudaMemcpyHostToDevice, st));
    // 3: T vector by a stable multisplit of each block's positions by byte
    {
      std::vector<int64_t> cb, c0(nvb + 1, 0);
      std::vector<int32_t> ci;
      for (int i = 0; i < nvb; ++i) {
        c0[i] = (int64_t)cb.size();
        for (int32_t k = 0; (int64_t)k * kTChunk < vb[i].n; ++k) {
          cb.push_back(i);
          ci.push_back(k);
        }
      }
      c0[nvb] = (int64_t)cb.size();
      const int64_t ntc = (int64_t)cb.size();
      BZD_TRY(g.vals2.ensure((size_t)tot * 4));
      BZD_TRY(g.tcb.ensure((size_t)std::max<int64_t>(ntc, 1) * 8));
      BZD_TRY(g.tci.ensure((size_t)std::max<int64_t>(ntc, 1) * 4));
      BZD_TRY(g.tc0.ensure((size_t)(nvb + 1) * 8));
      BZD_TRY(g.tcnt.ensure((size_t)std::max<int64_t>(ntc, 1) * 256 * 4));
      BZD_TRY(cudaMemcpyAsync(g.tcb.p, cb.data(), (size_t)ntc * 8, cudaMemcpyHostToDevice, st));
      BZD_TRY(cudaMemcpyAsync(g.tci.p, ci.data(), (size_t)ntc * 4, cudaMemcpyHostToDevice, st));
      BZD_TRY(cudaMemcpyAsync(g.tc0.p, c0.data(), (size_t)(nvb + 1) * 8, cudaMemcpyHostToDevice, st));
      if (ntc) {
        tchunk_count_kernel<<<(unsigned)ntc, 256, 0, st>>>(g.vb.as<VBlock>(), g.L.as<uint8_t>(), g.tcb.as<int64_t>(),
                                                           g.tci.as<int32_t>(), ntc, g.tcnt.as<uint32_t>());
        tchunk_offsets_kernel<<<nvb, 256, 0, st>>>(g.vb.as<VBlock>(), g.tc0.as<int64_t>(), g.tcnt.as<uint32_t>());
        tchunk_place_kernel<<<(unsigned)((ntc + 3) / 4), 128, 0, st>>>(g.vb.as<VBlock>(), g.L.as<uint8_t>(),
                                                                     g.tcb.as<int64_t>(), g.tci.as<int32_t>(), ntc,
                                                                     g.tcnt.as<uint32_t>(), g.vals2.as<uint32_t>());
      }
    }
    mark("sort");
    const uint32_t *T = g.vals2.as<uint32_t>();
    chain_start_kernel<<<(nvb + 255) / 256, 256, 0, st>>>(g.vb.as<VBlock>(), nvb, T);
    BZD_TRY(g.rblk.ensure((size_t)nr * 8));
    BZD_TRY(g.rnext.ensure((size_t)nr * 4));
    BZD_TRY(g.rlen.ensure((size_t)nr * 4));
    BZD_TRY(g.rrank.ensure((size_t)nr * 4));
    BZD_TRY(cudaMemcpyAsync(g.rblk.p, rblk.data(), (size_t)nr * 8, cudaMemcpyHostToDevice, st));
    ruler_walk_kernel<<<grid_of(nr), 256, 0, st>>>(g.vb.as<VBlock>(), nvb, T, g.rblk.as<int64_t>(), nr,
                                                  g.rnext.as<int32_t>(), g.rlen.as<int32_t>());
    ruler_rank_kernel<<<(nvb + 127) / 128, 128, 0, st>>>(g.vb.as<VBlock>(), nvb, g.rnext.as<int32_t>(),
                                                         g.rlen.as<int32_t>(), g.rrank.as<int32_t>());
    BZD_TRY(g.bwt.ensure((size_t)tot));
    ruler_write_kernel<<<grid_of(nr), 256, 0, st>>>(g.vb.as<VBlock>(), T, g.L.as<uint8_t>(), g.rblk.as<int64_t>(), nr,
                                                   g.rlen.as<int32_t>(), g.rrank.as<int32_t>(), g.bwt.as<uint8_t>());
    mark("list ranking");
    // 4: inverse RLE1: lengths, offsets on the host, bytes + CRCs
    rle1_kernel<false><<<(nvb + 3) / 4, 128, 0, st>>>(g.vb.as<VBlock>(), nvb, g.bwt.as<uint8_t>(), nullptr);
    BZD_TRY(cudaMemcpyAsync(vb.data(), g.vb.p, (size_t)nvb * sizeof(VBlock), cudaMemcpyDeviceToHost, st));
    BZD_TRY(cudaStreamSynchronize(st));
    for (int s = 0; s < ns; ++s) {
      if (!ok[s]) continue;
      int64_t o = out_off[ids[s]];
      for (int i = range[s].first; i < range[s].second; ++i) {
        if (vb[i].status) ok[s] = 0;
        vb[i].out_off = o;
        o += vb[i].out_len;
      }
      if (o - out_off[ids[s]] != out_len[ids[s]]) ok[s] = 0;
      if (!ok[s])
        for (int i = range[s].first; i < range[s].second; ++i) vb[i].status = 4;   // do not write
    }
    BZD_TRY(cudaMemcpyAsync(g.vb.p, vb.data(), (size_t)nvb * sizeof(VBlock), cudaMemcpyHostToDevice, st));
    rle1_kernel<true><<<(nvb + 3) / 4, 128, 0, st>>>(g.vb.as<VBlock>(), nvb, g.bwt.as<uint8_t>(), d_out);
    mark("rle1");
    {
      std::vector<int64_t> cb;
      std::vector<int32_t> cidx;
      for (int i = 0; i < nvb; ++i)
        if (!vb[i].status)
          for (int64_t k = 0; k * kCrcChunk < vb[i].out_len; ++k) {
            cb.push_back(i);
            cidx.push_back((int32_t)k);
          }
      const int64_t nch = (int64_t)cb.size();
      BZD_TRY(g.zs.ensure(40 * 32 * 4));
      if (!g.zs_ready) {
        // M^(2^k): image of every register bit after 2^k zero bytes
        std::vector<uint32_t> zs(40 * 32);
        auto step = [](uint32_t c) {
          for (int b = 0; b < 8; ++b) c = (c & 0x80000000u) ? (c << 1) ^ 0x04C11DB7u : (c << 1);
          return c;
        };
        for (int bit = 0; bit < 32; ++bit) zs[bit] = step(1u << bit);
        for (int k = 1; k < 40; ++k)
          for (int bit = 0; bit < 32; ++bit) {
            uint32_t v = zs[(k - 1) * 32 + bit], r = 0;
            for (int q = 0; q < 32; ++q)
              if (v & (1u << q)) r ^= zs[(k - 1) * 32 + q];
            zs[k * 32 + bit] = r;
          }
        // on the decode stream (a pageable cudaMemcpy is not ordered with it)
        BZD_TRY(cudaMemcpyAsync(g.zs.p, zs.data(), zs.size() * 4, cudaMemcpyHostToDevice, st));
        BZD_TRY(cudaStreamSynchronize(st));
        g.zs_ready = true;
      }
      BZD_TRY(g.crcacc.ensure((size_t)nvb * 4));
      BZD_TRY(cudaMemsetAsync(g.crcacc.p, 0, (size_t)nvb * 4, st));
      if (nch) {
        BZD_TRY(g.cblk.ensure((size_t)nch * 8));
        BZD_TRY(g.cidx.ensure((size_t)nch * 4));
        BZD_TRY(cudaMemcpyAsync(g.cblk.p, cb.data(), (size_t)nch * 8, cudaMemcpyHostToDevice, st));
        BZD_TRY(cudaMemcpyAsync(g.cidx.p, cidx.data(), (size_t)nch * 4, cudaMemcpyHostToDevice, st));
        crc_chunks_kernel<<<grid_of(nch, 128), 128, 0, st>>>(g.vb.as<VBlock>(), g.cblk.as<int64_t>(), g.cidx.as<int32_t>(),
                                                             nch, d_out, g.zs.as<uint32_t>(), g.crcacc.as<uint32_t>());
      }
      crc_finish_kernel<<<(nvb + 127) / 128, 128, 0, st>>>(g.vb.as<VBlock>(), nvb, g.zs.as<uint32_t>(),
                                                           g.crcacc.as<uint32_t>());
    }
    BZD_TRY(cudaMemcpyAsync(vb.data(), g.vb.p, (size_t)nvb * sizeof(VBlock), cudaMemcpyDeviceToHost, st));
    BZD_TRY(cudaStreamSynchronize(st));
    mark("rle1 + crc");
  }
  // CRCs: every block's, then the stream's combined CRC (bzlib.c)
  for (int s = 0; s < ns; ++s) {
    if (!ok[s]) continue;
    uint32_t comb = 0;
    for (int i = range[s].first; i < range[s].second; ++i) {
      if (vb[i].status || vb[i].crc != vb_crc[i]) { ok[s] = 0; break; }
      comb = ((comb << 1) | (comb >> 31)) ^ vb[i].crc;
    }
    if (ok[s] && comb != stored_comb[s]) ok[s] = 0;
    if (ok[s] && range[s].first == range[s].second && out_len[ids[s]] != 0) ok[s] = 0;
    if (ok[s]) status[ids[s]] = 0;
  }
  return 0;
}

}  // namespace

// Decode payloads[i] (plen[i] bytes, one bzip2 stream each) into d_out +
// out_off[i], expecting out_len[i] bytes.  status[i]: 0 decoded (or skipped
// by the caller: status[i] == 0 on entry is left alone), 1 = not decoded
// here (the caller decodes it with libbzip2).  Returns 0, or < 0 on a CUDA
// error (message in err).
int decode_payloads(const uint8_t *const *payloads, const int64_t *plen, int n, uint8_t *d_out,
                    const int64_t *out_off, const int64_t *out_len, uint8_t *status, cudaStream_t st,
                    std::string &err) {
  const int64_t kBatchBytes = (int64_t)1 << 30;   // compressed bytes per batch (bounds the L / sort buffers)
  std::vector<int> ids;
  int64_t acc = 0;
  for (int i = 0; i <= n; ++i) {
    if (i == n || (acc + (i < n ? plen[i] : 0) > kBatchBytes && !ids.empty())) {
      if (!ids.empty()) {
        const int rc = decode_batch(payloads, plen, ids, d_out, out_off, out_len, status, st, err);
        if (rc) return rc;
      }
      ids.clear();
      acc = 0;
      if (i == n) break;
    }
    if (status[i] == 0) continue;
    status[i] = 1;
    ids.push_back(i);
    acc += plen[i];
  }
  return 0;
}

}  // namespace bzd
}  // namespace pcbz
