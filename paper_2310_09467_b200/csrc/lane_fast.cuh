// lane_fast.cuh -- the hot loop of the judge: one lane's run of 8-pixel
// chunks (included by judge_kernel.cuh; needs ChainState, claim_word,
// ld/st/atom helpers from there; included inside namespace pcbz).
#pragma once


// rows of one 8-pixel chunk: X = row y, T1 = row y-1, TS = row y-py
struct ChunkRows {
  uint4 X, T1, TS;
};

// Branch-free chunk load: rows above the frame read as 0 (the reference's
// out-of-bounds neighbours, _kernels.py:33-35); TEMP forms (F - P) mod 2^16.
template <bool TEMP>
__device__ __forceinline__ uint4 ld_row(const uint16_t *__restrict__ s,
                                        const uint16_t *__restrict__ p, int64_t off, bool ok) {
  const int64_t o = ok ? off : 0;
  uint4 a = __ldg(reinterpret_cast<const uint4 *>(s + o));
  if constexpr (TEMP) {
    const uint4 b = __ldg(reinterpret_cast<const uint4 *>(p + o));
    a.x = sub16x2(a.x, b.x); a.y = sub16x2(a.y, b.y);
    a.z = sub16x2(a.z, b.z); a.w = sub16x2(a.w, b.w);
  }
  if (!ok) a = make_uint4(0, 0, 0, 0);
  return a;
}

template <bool TEMP, bool NT1, bool NTS>
__device__ __forceinline__ ChunkRows ld_chunk_rows(const uint16_t *s, const uint16_t *p, int W,
                                                   int py, int y, int x0) {
  const int64_t off = (int64_t)y * W + x0;
  ChunkRows c;
  c.X = ld_row<TEMP>(s, p, off, true);
  c.T1 = NT1 ? ld_row<TEMP>(s, p, off - W, y >= 1) : make_uint4(0, 0, 0, 0);
  c.TS = NTS ? ld_row<TEMP>(s, p, off - (int64_t)py * W, y >= py) : make_uint4(0, 0, 0, 0);
  return c;
}

// Left-neighbour history carried between chunks of one row (zero at a row start).
struct History {
  uint4 X1, X2, T1, S1, S2;  // X of chunks k-1, k-2; T1 of k-1; TS of k-1, k-2
};

// Residuals of the 8 pixels of a chunk for compile-time predictor ID and
// lenslet pitch PX (_kernels.py:46-66, 179-186).
template <int PX, int ID>
__device__ __forceinline__ void chunk_residuals8(const ChunkRows &c, const History &h,
                                                 uint32_t (&r)[8]) {
  constexpr int GRP = ID == 0 ? -1 : (ID - 1) / 4;
  constexpr int F = ID == 0 ? 0 : (ID - 1) % 4 + 1;
  constexpr bool kT1 = GRP == 0 || GRP == 2;
  constexpr bool kTS = GRP == 1 || GRP == 2;
  int X[8];
  unpack8(c.X, X);
  if constexpr (GRP < 0) {
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = (uint32_t)X[i];
    return;
  } else {
    int T1[8], TS[8], H1[8], H2[8], S1[8], S2[8], t1h[8];
    unpack8(h.X1, H1);
    if constexpr (kT1) { unpack8(c.T1, T1); unpack8(h.T1, t1h); }
    if constexpr (kTS) {
      unpack8(c.TS, TS); unpack8(h.S1, S1);
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
// returned word is claimed at the end of the chunk; the kernel sweeps once
// more after the loop for crossings nobody observed.
__device__ __forceinline__ void chunk_events(const ChainState &cs, const uint32_t (&r)[8],
                                             uint32_t &prev_lo) {
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
  for (int e = 0; e < 16; ++e) {
    const uint32_t la = cs.lbase + key[e] * 2u + (key[e] >> 1) * (4u * kJudgeThreads - 4u);
    last[e] = lds_u16(la);
    sts_u16(la, prd[e]);
  }
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
      if (last[e] == kUnseen) cs.F[key[e] * kJudgeThreads] = (uint8_t)prd[e];
  }
  if (flag & 0x80008000u) {  // some counter has crossed 0x8000: claim
#pragma unroll
    for (int e = 0; e < 16; ++e)
      if (word[e] < (uint32_t)kHistWords) claim_word(cs, word[e]);
  }
}

// Advance history past a chunk that ended at column x0 + 8.
template <int PX, int ID>
__device__ __forceinline__ void advance_history(History &h, const ChunkRows &c, bool row_end) {
  const uint4 Z = make_uint4(0, 0, 0, 0);
  if (row_end) {
    h.X1 = h.X2 = h.T1 = h.S1 = h.S2 = Z;  // next chunk starts a row: left neighbours are 0
  } else {
    h.X2 = h.X1; h.X1 = c.X; h.T1 = c.T1; h.S2 = h.S1; h.S1 = c.TS;
  }
}

// One lane's run of `nch` chunks starting at pixel a (a % 8 == 0).  Chunks are
// processed in pairs with the next pair's rows already in flight (explicit
// double buffering: the loads are consumed one pair later).
template <int PX, int ID, bool TEMP>
__device__ __noinline__ void lane_fast(const uint16_t *__restrict__ src,
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
  {  // history of a run that starts mid-row
    const int64_t off = (int64_t)y * W + x0;
    const int64_t offs = off - (int64_t)py * W;
    h.X1 = ld_row<TEMP>(src, prv, off - 8, GRP >= 0 && x0 >= 8);
    h.X2 = ld_row<TEMP>(src, prv, off - 16, kTS && PX > 8 && x0 >= 16);
    h.T1 = ld_row<TEMP>(src, prv, off - W - 8, kT1 && x0 >= 8 && y >= 1);
    h.S1 = ld_row<TEMP>(src, prv, offs - 8, kTS && x0 >= 8 && y >= py);
    h.S2 = ld_row<TEMP>(src, prv, offs - 16, kTS && PX > 8 && x0 >= 16 && y >= py);
  }
  // positions of chunks c (y, x0) and c + 1 (y1, x1)
  auto step = [&](int &yy, int &xx) {
    xx += 8;
    if (xx == W) { xx = 0; ++yy; }
  };
  int y1 = y, x1 = x0;
  step(y1, x1);
  const int64_t last_c = nch - 1;
  ChunkRows c0 = ld_chunk_rows<TEMP, kT1, kTS>(src, prv, W, py, y, x0);
  ChunkRows c1 = ld_chunk_rows<TEMP, kT1, kTS>(src, prv, W, py, nch > 1 ? y1 : y,
                                              nch > 1 ? x1 : x0);
  for (int64_t c = 0; c < nch; c += 2) {
    // rows of chunks c+2, c+3 (clamped to the run: never read past it)
    int y2 = y1, x2 = x1;
    step(y2, x2);
    int y3 = y2, x3 = x2;
    step(y3, x3);
    const bool has2 = c + 2 <= last_c, has3 = c + 3 <= last_c;
    const ChunkRows n0 = ld_chunk_rows<TEMP, kT1, kTS>(src, prv, W, py, has2 ? y2 : y,
                                                      has2 ? x2 : x0);
    const ChunkRows n1 = ld_chunk_rows<TEMP, kT1, kTS>(src, prv, W, py, has3 ? y3 : y,
                                                      has3 ? x3 : x0);
    uint32_t r[8];
    chunk_residuals8<PX, ID>(c0, h, r);
    chunk_events(cs, r, prev_lo);
    advance_history<PX, ID>(h, c0, x1 == 0);
    if (c + 1 <= last_c) {
      chunk_residuals8<PX, ID>(c1, h, r);
      chunk_events(cs, r, prev_lo);
      advance_history<PX, ID>(h, c1, x2 == 0);
    }
    y = y2; x0 = x2; y1 = y3; x1 = x3;
    c0 = n0; c1 = n1;
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

