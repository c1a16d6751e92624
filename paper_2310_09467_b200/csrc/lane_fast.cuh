// lane_fast.cuh -- the hot loop of the judge: one lane's run of 8-pixel
// chunks (included by judge_kernel.cuh inside namespace pcbz; uses
// ChainState, claim_word and the ld/st/atom helpers defined there).
#pragma once

// 16 zero bytes: rows above the frame are loaded from here (the reference's
// out-of-bounds neighbours read 0, _kernels.py:33-35), so no select ever
// waits on a load result.
static __device__ const uint4 g_zero_chunk = {0u, 0u, 0u, 0u};

// 128-bit read-only load whose position in the instruction stream is pinned
// (volatile asm is not sunk toward its use, so the next chunk's rows really
// are in flight while the current chunk is processed).
#ifndef PCBZ_LDG_HINT
#define PCBZ_LDG_HINT 0   // 1: L2::evict_last on the row loads (A/B of the DRAM re-reads)
#endif
__device__ __forceinline__ uint4 ldg_v4_pinned(const uint16_t *p) {
  uint4 r;
#if PCBZ_LDG_HINT == 1
  asm volatile("{\n\t.reg .b64 pol;\n\tcreatepolicy.fractional.L2::evict_last.b64 pol, 1.0;\n\t"
               "ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], pol;\n\t}"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
#else
  asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
#endif
  return r;
}

// Raw rows of one 8-pixel chunk: X = row y, T1 = row y-1, TS = row y-py
// (and the same rows of the previous frame for temporal candidates; the
// modular delta is formed when the chunk is consumed, not when it is loaded).
struct ChunkRows {
  uint4 X, T1, TS, pX, pT1, pTS;
};

#ifndef PCBZ_PREFETCH
#define PCBZ_PREFETCH 0   // L2 prefetch distance in chunks (0 = off)
#endif
__device__ __forceinline__ void prefetch_l2(const uint16_t *p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

template <bool TEMP, bool NT1, bool NTS>
__device__ __forceinline__ ChunkRows ld_chunk_rows(const uint16_t *s, const uint16_t *p, int W,
                                                   int py, int y, int x0) {
  const uint16_t *z = reinterpret_cast<const uint16_t *>(&g_zero_chunk);
  const int64_t off = (int64_t)y * W + x0;
  const int64_t o1 = off - W, os = off - (int64_t)py * W;
  if constexpr (PCBZ_PREFETCH > 0) {
    // the rows PCBZ_PREFETCH chunks ahead (the next lines of this lane's run);
    // DRAM misses then overlap the chunks in between
    const int64_t d = 8 * PCBZ_PREFETCH;
    prefetch_l2(s + off + d);
    if constexpr (NT1) prefetch_l2(s + (y >= 1 ? o1 : off) + d);
    if constexpr (NTS) prefetch_l2(s + (y >= py ? os : off) + d);
    if constexpr (TEMP) prefetch_l2(p + off + d);
  }
  ChunkRows c;
  c.X = ldg_v4_pinned(s + off);
  if constexpr (NT1) c.T1 = ldg_v4_pinned(y >= 1 ? s + o1 : z);
  if constexpr (NTS) c.TS = ldg_v4_pinned(y >= py ? s + os : z);
  if constexpr (TEMP) {
    c.pX = ldg_v4_pinned(p + off);
    if constexpr (NT1) c.pT1 = ldg_v4_pinned(y >= 1 ? p + o1 : z);
    if constexpr (NTS) c.pTS = ldg_v4_pinned(y >= py ? p + os : z);
  }
  return c;
}

// Row pointers of the chunk a lane loads next (PCBZ_INCPTR): advanced by
// one chunk per iteration instead of re-deriving y * W + x0 and the
// out-of-frame selects per chunk; rows above the frame point at the zero
// chunk with a zero step.  Re-derived only at a row change.
struct RowPtrs {
  const uint16_t *x, *t1, *ts, *px, *pt1, *pts;
  int d1, ds;  // element step of the T1 / TS rows: 8, or 0 on the zero chunk
};

template <bool TEMP, bool NT1, bool NTS>
__device__ __forceinline__ RowPtrs row_ptrs(const uint16_t *s, const uint16_t *p, int W, int py, int y,
                                            int x0) {
  const uint16_t *z = reinterpret_cast<const uint16_t *>(&g_zero_chunk);
  const int64_t off = (int64_t)y * W + x0;
  RowPtrs r;
  r.d1 = y >= 1 ? 8 : 0;
  r.ds = y >= py ? 8 : 0;
  r.x = s + off;
  r.t1 = NT1 && y >= 1 ? s + off - W : z;
  r.ts = NTS && y >= py ? s + off - (int64_t)py * W : z;
  if constexpr (TEMP) {
    r.px = p + off;
    r.pt1 = NT1 && y >= 1 ? p + off - W : z;
    r.pts = NTS && y >= py ? p + off - (int64_t)py * W : z;
  }
  return r;
}

template <bool TEMP, bool NT1, bool NTS>
__device__ __forceinline__ void advance(RowPtrs &r) {
  r.x += 8;
  if constexpr (NT1) r.t1 += r.d1;
  if constexpr (NTS) r.ts += r.ds;
  if constexpr (TEMP) {
    r.px += 8;
    if constexpr (NT1) r.pt1 += r.d1;
    if constexpr (NTS) r.pts += r.ds;
  }
}

template <bool TEMP, bool NT1, bool NTS>
__device__ __forceinline__ ChunkRows ld_ptrs(const RowPtrs &r) {
  ChunkRows c;
  c.X = ldg_v4_pinned(r.x);
  if constexpr (NT1) c.T1 = ldg_v4_pinned(r.t1);
  if constexpr (NTS) c.TS = ldg_v4_pinned(r.ts);
  if constexpr (TEMP) {
    c.pX = ldg_v4_pinned(r.px);
    if constexpr (NT1) c.pT1 = ldg_v4_pinned(r.pt1);
    if constexpr (NTS) c.pTS = ldg_v4_pinned(r.pts);
  }
  return c;
}

__device__ __forceinline__ uint4 sub16x2_4(const uint4 &a, const uint4 &b) {
  return make_uint4(sub16x2(a.x, b.x), sub16x2(a.y, b.y), sub16x2(a.z, b.z), sub16x2(a.w, b.w));
}

// source rows of a chunk: the frame, or (F - P) mod 2^16 (predictors.py:116-120)
template <bool TEMP, bool NT1, bool NTS>
__device__ __forceinline__ void source_rows(const ChunkRows &c, uint4 &X, uint4 &T1, uint4 &TS) {
  const uint4 Z = make_uint4(0, 0, 0, 0);
  if constexpr (TEMP) {
    X = sub16x2_4(c.X, c.pX);
    T1 = NT1 ? sub16x2_4(c.T1, c.pT1) : Z;
    TS = NTS ? sub16x2_4(c.TS, c.pTS) : Z;
  } else {
    X = c.X;
    T1 = NT1 ? c.T1 : Z;
    TS = NTS ? c.TS : Z;
  }
}

// Left-neighbour history carried between chunks of one row (zero at a row start).
struct History {
  uint4 X1, X2, T1, S1, S2;  // X of chunks k-1, k-2; T1 of k-1; TS of k-1, k-2
};

// Residuals of the 8 pixels of a chunk for compile-time predictor ID and
// lenslet pitch PX (_kernels.py:46-66, 179-186).
template <int PX, int ID>
__device__ __forceinline__ void chunk_residuals8(const uint4 &cX, const uint4 &cT1, const uint4 &cTS,
                                                 const History &h, uint32_t (&r)[8]) {
  constexpr int GRP = ID == 0 ? -1 : (ID - 1) / 4;
  constexpr int F = ID == 0 ? 0 : (ID - 1) % 4 + 1;
  constexpr bool kT1 = GRP == 0 || GRP == 2;
  constexpr bool kTS = GRP == 1 || GRP == 2;
  int X[8];
  unpack8(cX, X);
  if constexpr (GRP < 0) {
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = (uint32_t)X[i];
    return;
  } else {
    int T1[8], TS[8], H1[8], H2[8], S1[8], S2[8], t1h[8];
    unpack8(h.X1, H1);
    if constexpr (kT1) { unpack8(cT1, T1); unpack8(h.T1, t1h); }
    if constexpr (kTS) {
      unpack8(cTS, TS); unpack8(h.S1, S1);
      if constexpr (PX > 8) { unpack8(h.X2, H2); unpack8(h.S2, S2); }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int p = 0, p1 = 0;
      if constexpr (kT1) p1 = pred_f<F>(i ? X[i - 1] : H1[7], T1[i], i ? T1[i - 1] : t1h[7]);
      if constexpr (kTS) {
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

// The 16 events of one chunk (_kernels.py:187-202):
//   e = 2i: (hi_i, lo_{i-1})     e = 2i + 1: (lo_i, hi_i)
// Phase A performs the last-pred lookups/updates in stream order (independent
// 16-bit load + store each); phase B issues one unconditional shared atomic
// per event -- a first occurrence (last == 0x100, bin 0x100xx) lands in the
// dummy row past the histogram.  A counter found with bit 15 set in any
// returned word is claimed one chunk later (the returned words of chunk c are
// examined after chunk c+1's atomics are issued, so nothing waits on them);
// the kernel sweeps once more after the loop for crossings nobody observed.
//
// Deferred state of the previous chunk: its returned words and its words.
struct Pending {
  uint32_t old[16], word[16];
};

__device__ __forceinline__ void settle_pending(const ChainState &cs, const Pending &pd) {
  uint32_t flag = 0;
#pragma unroll
  for (int e = 0; e < 16; e += 2) flag |= pd.old[e] | pd.old[e + 1];
  if (flag & 0x80008000u) {  // some counter has crossed 0x8000: claim
#pragma unroll
    for (int e = 0; e < 16; ++e)
      if (pd.word[e] < (uint32_t)kHistWords) claim_word(cs, pd.word[e]);
  }
}

__device__ __forceinline__ void chunk_events(const ChainState &cs, const uint32_t (&r)[8],
                                             uint32_t &prev_lo, Pending &pd) {
  uint32_t key[16], prd[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    key[2 * i] = r[i] >> 8;
    prd[2 * i] = i ? (r[i - 1] & 0xFFu) : prev_lo;
    key[2 * i + 1] = r[i] & 0xFFu;
    prd[2 * i + 1] = r[i] >> 8;
  }
  // lt_code of both bytes of a residual at once: hi | lo << 16, one multiply
  // and one mask for the pair (13 * 255 < 2^16, so the halves never carry)
  uint32_t code[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t v2 = __byte_perm(r[i], 0, 0x4041);  // hi | lo << 16
    const uint32_t cp = (v2 << 7) | ((v2 * kSwizzleMul) & 0x007F007Fu);
    code[2 * i + 1] = cp & 0xFFFFu;               // lt_code(hi): pred of the lo event
    if (i < 7) code[2 * i + 2] = cp >> 16;        // lt_code(lo): pred of the next hi event
  }
  code[0] = lt_code(prev_lo);
  prev_lo = r[7] & 0xFFu;
  uint32_t last[16];  // last-pred codes (lt_code), kUnseenCode for a first occurrence
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const uint32_t la = cs.lbase + key[e] * (2u * kJudgeThreads);  // u16 [key][lane]
    last[e] = lds_u16(la);
    sts_u16(la, code[e]);
  }
  // the previous chunk's returned words arrived long ago; examining them
  // first frees their registers, so this chunk's atomics return straight
  // into the pending state (no copies that would wait on them)
#ifndef PCBZ_DEFER
#define PCBZ_DEFER 0
#endif
  if constexpr (PCBZ_DEFER) settle_pending(cs, pd);
  uint32_t fresh = 0;
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    fresh |= last[e];
    pd.word[e] = hist_word(last[e], prd[e]);  // bin = last * 256 + pred, 2 bins/word
    pd.old[e] = atoms_add(cs.hbase + 4u * pd.word[e], pred_inc(prd[e]));
  }
  if constexpr (!PCBZ_DEFER) {  // examine this chunk's returned words right away
    settle_pending(cs, pd);
#pragma unroll
    for (int e = 0; e < 16; ++e) pd.old[e] = 0;
  }
  if (fresh & kUnseenCode) {  // first occurrence of a key in this run
#pragma unroll
    for (int e = 0; e < 16; ++e)
      if (last[e] == kUnseenCode) cs.F[key[e] * kJudgeThreads] = (uint8_t)prd[e];
  }
}

// One lane's run of `nch` chunks starting at pixel a (a % 8 == 0).  The next
// chunk's rows are issued at the top of each iteration (pinned loads) and
// consumed one iteration later.
#ifndef PCBZ_LANE_INLINE
#define PCBZ_LANE_INLINE 0
#endif
#if PCBZ_LANE_INLINE
#define PCBZ_LANE_ATTR __forceinline__
#else
#define PCBZ_LANE_ATTR __noinline__
#endif
template <int PX, int ID, bool TEMP>
__device__ PCBZ_LANE_ATTR void lane_fast(const uint16_t *__restrict__ src,
                                       const uint16_t *__restrict__ prv, int W, int py,
                                       int64_t npix, int64_t a, int64_t nch, const PredCfg cfg,
                                       const ChainState cs) {
  constexpr int GRP = ID == 0 ? -1 : (ID - 1) / 4;
  constexpr bool kT1 = GRP == 0 || GRP == 2;
  constexpr bool kTS = GRP == 1 || GRP == 2;
  if (nch <= 0) return;
  const int64_t q = a > 0 ? a - 1 : npix - 1;  // wrap predecessor (_kernels.py:172-190)
  uint32_t prev_lo = residual_at(src, prv, W, (int)(q / W), (int)(q % W), cfg) & 0xFFu;
  int y = (int)(a / W), x0 = (int)(a % W);
  History h;
  {  // history of a run that starts mid-row (rare: plain loads)
    const uint4 Z = make_uint4(0, 0, 0, 0);
    const int64_t off = (int64_t)y * W + x0;
    const int64_t offs = off - (int64_t)py * W;
    auto row = [&](int64_t o, bool ok) -> uint4 {
      if (!ok) return Z;
      uint4 v = __ldg(reinterpret_cast<const uint4 *>(src + o));
      if constexpr (TEMP) v = sub16x2_4(v, __ldg(reinterpret_cast<const uint4 *>(prv + o)));
      return v;
    };
    h.X1 = row(off - 8, GRP >= 0 && x0 >= 8);
    h.X2 = row(off - 16, kTS && PX > 8 && x0 >= 16);
    h.T1 = row(off - W - 8, kT1 && x0 >= 8 && y >= 1);
    h.S1 = row(offs - 8, kTS && x0 >= 8 && y >= py);
    h.S2 = row(offs - 16, kTS && PX > 8 && x0 >= 16 && y >= py);
  }
  {
    // iteration c issues the rows of chunk c+1, then computes the residuals
    // and events of chunk c.  Measured alternatives, all slower on C2/C3
    // (profiles/r01_notes.md): rows two chunks ahead, a software pipeline
    // (residuals of c+1 beside the events of c), two chunks per iteration
    // with ping-pong pending atomics, lane_fast inlined into the kernel.
#ifndef PCBZ_INCPTR
#define PCBZ_INCPTR 0
#endif
#if PCBZ_INCPTR
    RowPtrs rp = row_ptrs<TEMP, kT1, kTS>(src, prv, W, py, y, x0);
    ChunkRows cur = ld_ptrs<TEMP, kT1, kTS>(rp);
#else
    ChunkRows cur = ld_chunk_rows<TEMP, kT1, kTS>(src, prv, W, py, y, x0);
#endif
    Pending pd;
#pragma unroll
    for (int e = 0; e < 16; ++e) { pd.old[e] = 0; pd.word[e] = ~0u; }
    for (int64_t c = 0; c < nch; ++c) {
      int y1 = y, x1 = x0 + 8;
      if (x1 == W) { x1 = 0; ++y1; }
      const bool more = c + 1 < nch;
#if PCBZ_INCPTR
      if (more) {
        if (x1 == 0 && (y1 == 1 || y1 == py)) rp = row_ptrs<TEMP, kT1, kTS>(src, prv, W, py, y1, 0);
        else advance<TEMP, kT1, kTS>(rp);   // rows are contiguous across a row change
      }
      const ChunkRows nxt = ld_ptrs<TEMP, kT1, kTS>(rp);
#else
      const ChunkRows nxt = ld_chunk_rows<TEMP, kT1, kTS>(src, prv, W, py, more ? y1 : y,
                                                         more ? x1 : x0);
#endif
      uint4 X, T1, TS;
      source_rows<TEMP, kT1, kTS>(cur, X, T1, TS);
      uint32_t r[8];
      chunk_residuals8<PX, ID>(X, T1, TS, h, r);
      chunk_events(cs, r, prev_lo, pd);
      if (x1 == 0) {
        h.X1 = h.X2 = h.T1 = h.S1 = h.S2 = make_uint4(0, 0, 0, 0);  // next chunk starts a row
      } else {
        h.X2 = h.X1; h.X1 = X; h.T1 = T1; h.S2 = h.S1; h.S1 = TS;
      }
      y = y1; x0 = x1;
      cur = nxt;
    }
    settle_pending(cs, pd);
    return;
  }
}

template <int PX, bool TEMP, int... IDs>
__device__ __forceinline__ void lane_fast_dispatch(int id, const uint16_t *src,
                                                   const uint16_t *prv, int W, int py,
                                                   int64_t npix, int64_t a, int64_t nch,
                                                   const PredCfg &cfg, const ChainState &cs,
                                                   std::integer_sequence<int, IDs...>) {
  ((id == IDs ? lane_fast<PX, IDs, TEMP>(src, prv, W, py, npix, a, nch, cfg, cs) : void()), ...);
}
