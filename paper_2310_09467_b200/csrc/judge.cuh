// judge.cuh -- device-side building blocks and launch plumbing of the B200
// entropy judge (reference: pkg/src/pcbz/_kernels.py, criterion.py).
#pragma once
#include <cstdint>
#include <string>
#include <cuda_runtime.h>

namespace pcbz {

// ---- tunables ------------------------------
constexpr int kJudgeThreads = 192;             // lane-private chains per CTA (6 warps)
constexpr int kHistWords = 32768;              // 65536 packed u16 bins
constexpr int kDummyWords = 128;               // row 0x100xx: first occurrences land here
constexpr int kLastWords = 128;                // 256 keys x u16 per lane, 2 per word
constexpr uint32_t kUnseen = 0x100;            // per-lane "key not seen yet" marker
constexpr uint32_t kSpill = 0x8000;            // u16 bin spill threshold
constexpr int kSpillCap = 512;                 // spill list entries per CTA
constexpr int64_t kMaxSegPixels = 8000000;     // 2 events/pixel / kSpill < kSpillCap
constexpr int64_t kMinItemPixels = 1 << 18;    // smaller work items lose to per-item overhead
constexpr int kEntropyThreads = 192;           // all entropy reductions use this shape
constexpr int kMaxFastPitch = 16;              // fast path: pitch_x <= 16 (template parameter)
constexpr int kTermTable = 65536;              // precomputed entropy terms per call (entropy.cuh)
#ifndef PCBZ_TRACE_WORDS
#define PCBZ_TRACE_WORDS 3   // per-item trace stamps (5: + claim-sweep and stitch ends, for profiling)
#endif
constexpr int kTraceWords = PCBZ_TRACE_WORDS;
// per-item partial histogram of a multi-segment / band judge: the item's
// packed u16 words as they sit in shared memory, its spill count and its
// spilled bins (each + kSpill), written with plain stores (judge_kernel.cuh)
constexpr int kPartSpill = kHistWords;         // word index of the spill count
constexpr int kPartWords = kHistWords + 4 + kSpillCap;   // 16-byte multiple

constexpr size_t kJudgeSmemBytes =
    (size_t)(kHistWords + kDummyWords + kLastWords * kJudgeThreads + kSpillCap) * sizeof(uint32_t);

// One predictor's neighbourhood configuration; reference _kernels.py:56-59,167-170.
struct PredCfg {
  int f;    // prediction function 1..4 (0 = identity)
  int grp;  // -1 identity, 0 pixel-adjacent, 1 lenslet-stride, 2 phase (average)
  int sx, sy, px, py;
};

__host__ __device__ inline PredCfg make_cfg(int intra_id, int px, int py) {
  PredCfg c;
  c.px = px; c.py = py;
  if (intra_id == 0) { c.f = 0; c.grp = -1; c.sx = 1; c.sy = 1; return c; }
  c.f = (intra_id - 1) % 4 + 1;
  c.grp = (intra_id - 1) / 4;
  c.sx = c.grp == 0 ? 1 : px;
  c.sy = c.grp == 0 ? 1 : py;
  return c;
}

// Candidate lists of a batched judge call.  Frame 0 uses list A, frames >= 1
// list B (pipeline.py:67-73: temporal specs only where a previous frame exists).
struct CandLists {
  int k;                 // full candidate count (output row length)
  int kA, kB;
  uint8_t byteA[32], idxA[32];
  uint8_t byteB[32], idxB[32];
  // dispatch order of each list (positions, most expensive candidate first)
  // so the tail of the dynamic schedule holds the cheapest items
  uint8_t ordA[32], ordB[32];
};

struct JudgeParams {
  const uint16_t *frames;   // [nframes][npix]
  const uint16_t *halo;     // previous original frame of frames[0] or nullptr
  const uint16_t *delta;    // [nframes][npix] (F - P) mod 2^16 for temporal pairs, or nullptr
                            // (then formed in registers from both frames' rows)
  int64_t nframes, npix;
  int H, W, px, py;
  CandLists cl;
  int64_t npairs;           // scored (frame, candidate) pairs
  int S;                    // segments per pair (per band)
  int band, nbands;         // this call's band of a stream cut into nbands * S segments
  int64_t nslots;           // nframes * k (segment-summary stride of one band)
  int direct;               // 1: S == 1 and no histogram output -> entropy in-CTA
  int fast_px;              // >0: 8-pixel chunk path instantiated for pitch_x; 0: generic
  int lone_weight;          // run-length weight (x16) of warps alone on a scheduler
  double *ent;              // [nframes][k] (NaN = not scored)
  const double *terms;      // [nterms] entropy terms of this call's total (entropy.cuh)
  int64_t nterms;           // kTermTable (device table) or total + 1 (host-registered table)
  uint32_t *ghist;          // [nframes*k][65536] when !direct (summed over segments)
  uint32_t *part;           // [items][kPartWords] per-item partial histograms when !direct
  int64_t slot0, slot_count;  // slot-range finalize (owner-computes band merge): slots
                              // [slot0, slot0 + slot_count); slot_count 0 = per-pair mode
  int16_t *segsum;          // [nbands][nframes*k][S][2][256] when !direct
  // peer exchange of the band merge (pcbz_judge_merge_peers_device; nullptr
  // otherwise): device arrays of nbands pointers into every band's buffers,
  // mapped into this process (NVLink peer memory / symmetric memory)
  const uint64_t *peer_hist;  // [nbands] -> partial histograms [nbands*q][65536] u32
  const uint64_t *peer_summ;  // [nbands] -> segment summaries [nbands*q][S][2][256] i16
  const uint64_t *peer_ent;   // [nbands] -> gathered entropies [nbands*q] f64
  uint8_t *fscratch;        // [gridDim.x][kJudgeThreads][256]
  int *counter;             // dynamic item counter (zeroed before launch)
  uint64_t *trace;          // optional [items][3]: (smid << 48 | start ns, runs-done ns, end ns)
  int *err;                 // sticky error flag
};

struct EmitParams {
  const uint16_t *frames, *halo;
  int64_t nframes, npix;
  int H, W, px, py;
  const uint8_t *sel;       // [nframes] selected predictor byte
  uint8_t *stream;          // [nframes][2*(pix1-pix0)] big-endian residual bytes
  int64_t pix0, pix1;       // emitted pixel range of every frame (a band; 0, npix = all)
};

// launchers (judge.cu)
cudaError_t launch_judge(const JudgeParams &p, int grid, cudaStream_t st);
cudaError_t launch_finalize(const JudgeParams &p, cudaStream_t st);
// sum every scored slot's S item partials (+ spills) into ghist[slot], zero
// rows for unscored slots
cudaError_t launch_reduce_parts(const JudgeParams &p, cudaStream_t st);
// finalize of slots [p.slot0, p.slot0 + p.slot_count) (one block per slot)
cudaError_t launch_finalize_slots(const JudgeParams &p, cudaStream_t st);
cudaError_t launch_select(const JudgeParams &p, uint8_t *sel, cudaStream_t st);
// cross-rank flag barrier over peer memory: mode 1 arrive (store `epoch` at
// index `rank` of every peer's flag array), 2 wait (until every entry of
// this rank's array reached `epoch`), 3 both
cudaError_t launch_peer_signal(const uint64_t *peer_flags, uint32_t *my_flags, int nranks, int rank,
                               uint32_t epoch, int mode, cudaStream_t st);
cudaError_t launch_emit(const EmitParams &p, cudaStream_t st);       // per pixel, any shape
cudaError_t launch_emit_any(const EmitParams &p, cudaStream_t st);   // chunked when possible
cudaError_t launch_residual_image(const uint16_t *img, const uint16_t *prev, int64_t h, int64_t w,
                                  int spec, int px, int py, uint16_t *out, int big_endian,
                                  cudaStream_t st);
cudaError_t launch_temporal_delta(const uint16_t *cur, const uint16_t *prev, int64_t n,
                                  uint16_t *out, cudaStream_t st);
// delta[f][p] = frames[f][p] - prev(f)[p] mod 2^16 for f in [f0, nframes),
// p in [pix0, pix1) (8-aligned; prev(0) = halo)
cudaError_t launch_delta_frames(const uint16_t *frames, const uint16_t *halo, int64_t nframes,
                                int64_t npix, int64_t f0, int64_t pix0, int64_t pix1, uint16_t *delta,
                                cudaStream_t st);
cudaError_t launch_pair_hist(const uint8_t *s, int64_t n, uint32_t *hist, cudaStream_t st);
cudaError_t launch_counting_bwt(const uint8_t *s, int64_t n, uint8_t *out, uint32_t *scratch,
                                size_t scratch_words, cudaStream_t st);
size_t counting_bwt_scratch_words(int64_t n);
cudaError_t launch_term_table(double total, double *terms, cudaStream_t st);
cudaError_t launch_entropy_u64(const uint64_t *counts, double total, const double *terms,
                               int64_t nterms, double *out, cudaStream_t st);
// host-registered entropy term table of `total` on the current device (capi.cu), or nullptr
const double *registered_terms(int64_t total, int64_t *nterms);
cudaError_t launch_reconstruct(const uint16_t *res, const uint16_t *halo, int64_t nframes,
                               int64_t h, int64_t w, int px, int py, const uint8_t *sel,
                               uint16_t *out, cudaStream_t st);
cudaError_t judge_configure();  // one-time smem attribute setup

namespace bz {  // bzip2.cu
int compress_jobs(const uint8_t *d_in, const int64_t *in_off, int njobs, uint8_t *d_out, size_t out_cap,
                  int64_t *out_start, int64_t *out_len, uint8_t *host_needed, cudaStream_t st);
size_t job_bound(int64_t len);
const char *last_error();
}  // namespace bz

namespace bzd {  // bunzip2.cu
int decode_payloads(const uint8_t *const *payloads, const int64_t *plen, int n, uint8_t *d_out,
                    const int64_t *out_off, const int64_t *out_len, uint8_t *status, cudaStream_t st,
                    std::string &err);
cudaError_t launch_be16(const uint8_t *s, int64_t n, uint16_t *out, cudaStream_t st);
}  // namespace bzd

}  // namespace pcbz
