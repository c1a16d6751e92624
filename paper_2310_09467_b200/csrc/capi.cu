// capi.cu -- extern "C" boundary of libpcbz_b200.so (declared in
// include/pcbz_b200.h).  Host-buffer entry points stage data through a
// thread-local context (own stream + grow-only device buffers) so they are
// reentrant, like the reference's nogil kernels called from a ThreadPool
// (reference criterion.py:165-169, _kernels.py:157).
#include <cmath>
#include <cstdarg>
#include <thread>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pcbz_b200.h"
#include "judge.cuh"

using namespace pcbz;

namespace {

thread_local std::string g_err;
thread_local bool g_profile = false;
thread_local int g_launches = 0;
// CUDA events of profiled judge calls, summed lazily by pcbz_last_timing
struct TimedCall { cudaEvent_t e0, e1, e2; int launches; };
thread_local std::vector<TimedCall> g_timed;
thread_local int g_seg_override = 0;
thread_local bool g_fast_enabled = true;
// per-item trace of the last profiled judge (tools/trace_items.py)
thread_local bool g_trace_on = false;
thread_local uint64_t *g_trace_dev = nullptr;
thread_local size_t g_trace_cap = 0;
thread_local int64_t g_trace_items = 0;
thread_local int g_trace_segments = 0;

int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(x)                                                                    \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess)                                                             \
      return fail(PCBZ_E_CUDA, "%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_),    \
                  __FILE__, __LINE__);                                                 \
  } while (0)

int num_sms_cached() {
  static int nsm = -1;
  if (nsm < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) nsm = 148;
  }
  return nsm;
}

int check_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    return fail(PCBZ_E_NODEVICE, "no CUDA device visible");
  int dev = 0, major = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10) return fail(PCBZ_E_NODEVICE, "device %d is sm_%d x, this build is sm_100a", dev, major);
  static bool configured = false;
  if (!configured) {
    CUDA_TRY(judge_configure());
    configured = true;
  }
  return PCBZ_OK;
}

// grow-only device allocation
struct DevBuf {
  void *p = nullptr;
  size_t cap = 0;
  int ensure(size_t n) {
    if (n <= cap) return PCBZ_OK;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(n, 1 << 16);
    CUDA_TRY(cudaMalloc(&p, want));
    cap = want;
    return PCBZ_OK;
  }
  template <typename T> T *as() const { return reinterpret_cast<T *>(p); }
};

struct HostCtx {
  cudaStream_t stream = nullptr;
  cudaStream_t s_in = nullptr, s_out = nullptr;  // pcbz_judge_host copy streams
  cudaStream_t s_comp2 = nullptr;                // its second compute stream
  std::vector<cudaStream_t> s_more;              // further compute streams (PCBZ_HOST_STREAMS)
  DevBuf frames, prev, out, ent, sel, stream_out, hist, ws, scratch, bytes;
  int init() {
    if (stream) return PCBZ_OK;
    int rc = check_device();
    if (rc) return rc;
    CUDA_TRY(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    return PCBZ_OK;
  }
};

thread_local HostCtx g_ctx;

// Host-registered entropy term tables (pcbz_register_entropy_terms), one per
// (device, total), process-wide and never freed (a kernel enqueued by any
// thread may still read one), within a memory budget.
struct TermTable {
  int dev;
  int64_t total;
  double *d;
};
std::mutex g_terms_mu;
std::vector<TermTable> g_terms;
size_t g_terms_bytes = 0;

size_t terms_budget() {
  static const size_t b = [] {
    const char *e = getenv("PCBZ_TERMS_BUDGET_MB");
    return (size_t)(e ? atoll(e) : 4096) << 20;
  }();
  return b;
}

int validate_geometry(int64_t h, int64_t w, int64_t px, int64_t py) {
  if (h < 1 || w < 1) return fail(PCBZ_E_INVALID, "frame must contain at least one sample (h=%lld w=%lld)", (long long)h, (long long)w);
  if (px < 1 || py < 1) return fail(PCBZ_E_INVALID, "pitch must be positive (px=%lld py=%lld)", (long long)px, (long long)py);
  if (w > 0x7FFFFFFF || h > 0x7FFFFFFF || px > 0x7FFFFFFF || py > 0x7FFFFFFF)
    return fail(PCBZ_E_INVALID, "dimension exceeds int32");
  return PCBZ_OK;
}

int validate_specs(const uint8_t *specs, int k) {
  if (k < 1 || k > PCBZ_MAX_CANDIDATES) return fail(PCBZ_E_INVALID, "candidate count %d outside [1, %d]", k, PCBZ_MAX_CANDIDATES);
  for (int i = 0; i < k; ++i) {
    if ((specs[i] & 0x7F) > 12) return fail(PCBZ_E_INVALID, "invalid intra predictor id %d in byte 0x%02X", specs[i] & 0x7F, specs[i]);
    if (i && specs[i] <= specs[i - 1]) return fail(PCBZ_E_INVALID, "candidate bytes must be distinct and sorted ascending");
  }
  return PCBZ_OK;
}

// Work decomposition: segments per (frame, candidate) stream.  Items are
// pulled dynamically by one CTA per SM; item costs differ by candidate (up to
// ~1.8x, temporal phase predictors dearest; dispatched dearest first), and
// every extra segment adds a partial flush, a stitch and the merge.
// Measured (profiles/r01_notes.md, profiles/r02_band_sweep.jsonl,
// profiles/r02_sweep_c5.jsonl):
//  * small jobs (even the finest split is under two waves): fill one wave as
//    exactly as possible (C1, 13 pairs of 2048^2: S = 11, 143 items);
//  * whole frames with >= 8 waves unsplit: S = 1, direct mode (no flush or
//    merge; C2 1300 pairs, C3 2600);
//  * otherwise the fewest power-of-two segments giving items of <= ~2.2 M
//    pixels and >= 4 waves: every measured optimum -- 26 C2 frames S = 2
//    (42.3 vs 37.9 / 40.9 GB/s at S = 1 / 4), C4 S = 8 (13.0 vs 13.9 ms at 4),
//    C4 bands: 2 -> S = 4 (6.19 vs 6.55 / 7.21 ms), 4 -> S = 4 (3.24 vs
//    3.64 / 3.97), 8 -> S = 4 (1.90 vs 1.84 at S = 2, 2.26 at 8).
// Items stay >= kMinItemPixels, below which per-item overhead dominates.
int choose_segments(int64_t npairs, int64_t npix, bool want_hist, bool band = false) {
  (void)want_hist;
  auto env = [](const char *name, int64_t dflt) {
    const char *e = getenv(name);
    const int64_t v = e ? atoll(e) : dflt;
    return v < 1 ? 1 : v;
  };
  static const int64_t direct_waves = env("PCBZ_TARGET_WAVES", 8);
  static const int64_t min_waves = env("PCBZ_MIN_WAVES", 4);
  static const int64_t item_pixels = env("PCBZ_ITEM_PIXELS", 2200000);
  const int64_t nsm = num_sms_cached();
  const int64_t s_min = std::max<int64_t>(1, (npix + kMaxSegPixels - 1) / kMaxSegPixels);
  const int64_t s_cap = std::max<int64_t>(s_min, std::min<int64_t>(4096, npix / kMinItemPixels));
  if (npairs * s_cap < 2 * nsm) {
    int64_t best = s_min;
    double best_eff = -1.0;
    for (int64_t s = s_min; s <= s_cap; ++s) {
      const int64_t items = npairs * s;
      const double eff = (double)items / (double)(((items + nsm - 1) / nsm) * nsm);
      if (eff > best_eff + 1e-9) { best_eff = eff; best = s; }
    }
    return (int)best;
  }
  int64_t s = 1;
  while (s < s_min) s <<= 1;
  if (!band && s == 1 && npairs >= direct_waves * nsm) return 1;
  while ((npix / s > item_pixels || npairs * s < min_waves * nsm) && 2 * s <= s_cap) s <<= 1;
  return (int)std::max<int64_t>(s_min, std::min<int64_t>(s, s_cap));
}

struct Plan {
  JudgeParams jp{};
  int grid = 0;
  size_t ws_bytes = 0;
  size_t off_counter = 0, off_err = 0, off_terms = 0, off_fscratch = 0, off_segsum = 0, off_ghist = 0,
         off_part = 0;
};

// Relative cost class of scoring one predictor byte (per-item trace,
// profiles/r01_notes.md): temporal specs load two frames, the phase group
// three neighbourhoods; identity is cheapest.
int cost_class(uint8_t b) {
  const int id = b & 0x7F;
  const int grp = id == 0 ? 0 : 1 + (id - 1) / 4;  // 0 identity, 1 pixel, 2 lenslet, 3 phase
  return (b & 0x80 ? 4 : 0) + grp;
}

void order_by_cost(const uint8_t *bytes, int n, uint8_t *ord) {
  for (int i = 0; i < n; ++i) ord[i] = (uint8_t)i;
  std::stable_sort(ord, ord + n, [&](uint8_t a, uint8_t b) { return cost_class(bytes[a]) > cost_class(bytes[b]); });
}

int build_lists(const uint8_t *specs, int k, bool halo, int temporal, CandLists &cl) {
  memset(&cl, 0, sizeof cl);
  cl.k = k;
  for (int i = 0; i < k; ++i) {
    const bool t = specs[i] & 0x80;
    if (!t || (temporal && halo)) { cl.byteA[cl.kA] = specs[i]; cl.idxA[cl.kA++] = (uint8_t)i; }
    if (!t || temporal) { cl.byteB[cl.kB] = specs[i]; cl.idxB[cl.kB++] = (uint8_t)i; }
  }
  if (cl.kA == 0) return fail(PCBZ_E_INVALID, "no usable candidate for a frame without a previous frame");
  order_by_cost(cl.byteA, cl.kA, cl.ordA);
  order_by_cost(cl.byteB, cl.kB, cl.ordB);
  return PCBZ_OK;
}

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

// entropy terms of a plan: the host's table for this total if registered,
// else the per-call device table of the first kTermTable counts
// (term_table_kernel; larger counts evaluated inline)
bool use_registered_terms(JudgeParams &jp) {
  int64_t nt = 0;
  const double *t = registered_terms(2 * jp.npix - 1, &nt);
  if (!t) return false;
  jp.terms = t;
  jp.nterms = nt;
  return true;
}

// Run-length weight (in 1/16) of the two warps that own a scheduler alone
// (judge_kernel.cuh); tunable through PCBZ_LONE_WEIGHT for measurements.
int lone_weight() {
  static int w = [] {
    const char *e = getenv("PCBZ_LONE_WEIGHT");
    const int v = e ? atoi(e) : 16;  // equal runs measured best (profiles/r01_notes.md)
    return v < 8 ? 8 : (v > 64 ? 64 : v);
  }();
  return w;
}

// workspace offsets of a plan whose S / direct are set
void layout_workspace(Plan &pl, int64_t nframes, int k, bool want_hist) {
  const JudgeParams &jp = pl.jp;
  const int64_t items = jp.npairs * jp.S;
  pl.grid = (int)std::min<int64_t>(items, num_sms_cached());
  size_t off = 0;
  pl.off_counter = off; off = align_up(off + 4);
  pl.off_err = off; off = align_up(off + 4);
  pl.off_terms = off; off = align_up(off + (jp.nbands > 1 ? 0 : kTermTable * sizeof(double)));
  pl.off_fscratch = off; off = align_up(off + (size_t)pl.grid * kJudgeThreads * 256);
  if (!jp.direct) {
    // band calls keep the summaries in caller memory
    const size_t sums = jp.nbands > 1 ? 0 : (size_t)nframes * k * jp.S * 512 * sizeof(int16_t);
    pl.off_segsum = off; off = align_up(off + sums);
    pl.off_ghist = off; off = align_up(off + (want_hist ? 0 : (size_t)nframes * k * 65536 * 4));
    pl.off_part = off; off = align_up(off + (size_t)items * kPartWords * sizeof(uint32_t));
  }
  pl.ws_bytes = off;
}

// sched_pairs: pairs competing for the SMs when the segment count is chosen
// (0 = this plan's own; the chunked host pipeline passes the whole call's,
// since consecutive chunks overlap on two compute streams)
int make_plan(int64_t nframes, int64_t h, int64_t w, int64_t px, int64_t py, const uint8_t *specs,
              int k, bool halo, int temporal, bool want_hist, Plan &pl, int nbands = 1,
              int band = 0, int64_t sched_pairs = 0) {
  int rc = validate_geometry(h, w, px, py);
  if (rc) return rc;
  rc = validate_specs(specs, k);
  if (rc) return rc;
  if (nframes < 1) return fail(PCBZ_E_INVALID, "at least one frame is required");
  JudgeParams &jp = pl.jp;
  rc = build_lists(specs, k, halo, temporal, jp.cl);
  if (rc) return rc;
  jp.nframes = nframes;
  jp.npix = h * w;
  jp.H = (int)h; jp.W = (int)w; jp.px = (int)px; jp.py = (int)py;
  jp.npairs = jp.cl.kA + (nframes - 1) * jp.cl.kB;
  if (nbands < 1 || band < 0 || band >= nbands || nbands > jp.npix)
    return fail(PCBZ_E_INVALID, "band %d of %d invalid for %lld pixels", band, nbands, (long long)jp.npix);
  jp.band = band;
  jp.nbands = nbands;
  jp.nslots = nframes * k;
  const int64_t band_pix = (jp.npix + nbands - 1) / nbands;
  jp.S = g_seg_override > 0 ? (int)std::min<int64_t>(g_seg_override, band_pix)
                            : choose_segments(sched_pairs > 0 ? sched_pairs : jp.npairs, band_pix, want_hist,
                                              nbands > 1);
  if ((jp.npix + (int64_t)jp.S * nbands - 1) / ((int64_t)jp.S * nbands) > kMaxSegPixels)
    return fail(PCBZ_E_INVALID, "segment override %d leaves segments above %lld pixels", jp.S,
                (long long)kMaxSegPixels);
  jp.direct = (jp.S == 1 && nbands == 1 && !want_hist) ? 1 : 0;
  // 8-pixel chunk path: rows of whole chunks and a pitch the fast kernel is
  // instantiated for (pointer alignment is re-checked in run_plan)
  jp.fast_px = (w % 8 == 0 && px <= kMaxFastPitch && g_fast_enabled) ? (int)px : 0;
  jp.lone_weight = lone_weight();
  layout_workspace(pl, nframes, k, want_hist);
  return PCBZ_OK;
}

// Workspace bytes of any plan of this shape: the segment count depends on
// how many (frame, candidate) pairs are scored, which depends on the
// candidate lists (temporal specs are not scored on a halo-less frame 0), so
// take the maximum over every list size.
size_t workspace_upper_bound(int64_t nframes, int64_t h, int64_t w, int k, bool want_hist,
                             int nbands) {
  const int64_t npix = h * w;
  const int64_t band_pix = (npix + nbands - 1) / nbands;
  size_t best = 0;
  for (int ka = 1; ka <= k; ++ka)
    for (int kb = ka; kb <= k; ++kb) {
      Plan pl;
      JudgeParams &jp = pl.jp;
      jp.npairs = ka + (nframes - 1) * kb;
      jp.nbands = nbands;
      jp.S = g_seg_override > 0 ? (int)std::min<int64_t>(g_seg_override, band_pix)
                                : choose_segments(jp.npairs, band_pix, want_hist, nbands > 1);
      jp.direct = (jp.S == 1 && nbands == 1 && !want_hist) ? 1 : 0;
      layout_workspace(pl, nframes, k, want_hist);
      best = std::max(best, pl.ws_bytes);
    }
  return best;
}

// PCBZ_DELTA=0 keeps the in-register (F - P) of both frames' rows
bool use_delta(const JudgeParams &jp, const uint16_t *d_frames, const uint16_t *d_halo, bool band = false) {
  static const bool on = [] {
    const char *e = getenv("PCBZ_DELTA");
    return !(e && atoi(e) == 0);
  }();
  if (!on || (jp.nbands != 1 && !band) || jp.npix % 8 != 0) return false;
  if ((reinterpret_cast<uintptr_t>(d_frames) | reinterpret_cast<uintptr_t>(d_halo)) & 15) return false;
  for (int i = 0; i < jp.cl.kB; ++i)
    if (jp.cl.byteB[i] & 0x80) return true;
  for (int i = 0; i < jp.cl.kA; ++i)
    if (jp.cl.byteA[i] & 0x80) return true;
  return false;
}

// Stream-ordered scratch from the device's default pool; up to 2 GiB of it
// stays cached between calls (release threshold raised once per device),
// larger reservations go back to the driver at the next synchronisation.
cudaError_t pooled_alloc(void **p, size_t bytes, cudaStream_t st) {
  static bool configured[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 64 && !configured[dev]) {
    cudaMemPool_t pool;
    if ((e = cudaDeviceGetDefaultMemPool(&pool, dev)) != cudaSuccess) return e;
    uint64_t keep = 2ull << 30;
    if ((e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep)) != cudaSuccess) return e;
    configured[dev] = true;
  }
  return cudaMallocAsync(p, bytes, st);
}

// Enqueue the whole judge (+ optional emission) on `st`.
int run_plan(Plan &pl, const uint16_t *d_frames, const uint16_t *d_halo, double *d_ent,
             uint8_t *d_sel, uint8_t *d_stream, uint32_t *d_hist, void *d_ws, cudaStream_t st,
             int *d_err_shared = nullptr) {
  JudgeParams &jp = pl.jp;
  char *ws = static_cast<char *>(d_ws);
  jp.frames = d_frames;
  jp.halo = d_halo;
  if ((reinterpret_cast<uintptr_t>(d_frames) | reinterpret_cast<uintptr_t>(d_halo)) & 15)
    jp.fast_px = 0;  // 128-bit loads need 16-byte aligned frames
  jp.ent = d_ent;
  jp.counter = reinterpret_cast<int *>(ws + pl.off_counter);
  // a caller running several plans can collect all error flags in one word
  jp.err = d_err_shared ? d_err_shared : reinterpret_cast<int *>(ws + pl.off_err);
  jp.fscratch = reinterpret_cast<uint8_t *>(ws + pl.off_fscratch);
  jp.terms = reinterpret_cast<const double *>(ws + pl.off_terms);
  jp.nterms = kTermTable;
  const bool host_terms = use_registered_terms(jp);
  if (!jp.direct) {
    jp.segsum = reinterpret_cast<int16_t *>(ws + pl.off_segsum);
    jp.ghist = d_hist ? d_hist : reinterpret_cast<uint32_t *>(ws + pl.off_ghist);
    jp.part = reinterpret_cast<uint32_t *>(ws + pl.off_part);
  }
  TimedCall tc{nullptr, nullptr, nullptr, 0};
  if (g_profile) {
    cudaEventCreate(&tc.e0); cudaEventCreate(&tc.e1); cudaEventCreate(&tc.e2);
    cudaEventRecord(tc.e0, st);
  }
  int launches = 0;
  jp.trace = nullptr;
  if (g_trace_on) {
    const int64_t items = jp.npairs * jp.S;
    if ((size_t)items * kTraceWords > g_trace_cap) {
      if (g_trace_dev) cudaFree(g_trace_dev);
      g_trace_cap = 0;
      CUDA_TRY(cudaMalloc(&g_trace_dev, (size_t)items * 8 * kTraceWords));
      g_trace_cap = (size_t)items * kTraceWords;
    }
    jp.trace = g_trace_dev;
    g_trace_items = items;
    g_trace_segments = jp.S;
  }
  CUDA_TRY(cudaMemsetAsync(ws, 0, pl.off_terms, st));   // counter + err
  if (!host_terms) {
    CUDA_TRY(launch_term_table((double)(2 * jp.npix - 1), reinterpret_cast<double *>(ws + pl.off_terms), st));
    ++launches;
  }
  CUDA_TRY(cudaMemsetAsync(d_ent, 0xFF, (size_t)jp.nframes * jp.cl.k * sizeof(double), st));  // NaN
  // temporal candidates read a materialised delta frame (one pass per frame)
  // instead of both frames' rows per (frame, candidate) item
  uint16_t *d_delta = nullptr;
  jp.delta = nullptr;
  const int64_t delta_f0 = d_halo ? 0 : 1;
  if (use_delta(jp, d_frames, d_halo) && jp.nframes > delta_f0) {
    CUDA_TRY(pooled_alloc(reinterpret_cast<void **>(&d_delta), (size_t)jp.nframes * jp.npix * 2, st));
    CUDA_TRY(launch_delta_frames(d_frames, d_halo, jp.nframes, jp.npix, delta_f0, 0, jp.npix, d_delta, st));
    jp.delta = d_delta;
    ++launches;
  }
  CUDA_TRY(launch_judge(jp, pl.grid, st));
  ++launches;
  if (d_delta) CUDA_TRY(cudaFreeAsync(d_delta, st));
  if (!jp.direct) { CUDA_TRY(launch_reduce_parts(jp, st)); ++launches; }
  if (g_profile) cudaEventRecord(tc.e1, st);
  if (!jp.direct) { CUDA_TRY(launch_finalize(jp, st)); ++launches; }
  CUDA_TRY(launch_select(jp, d_sel, st));
  ++launches;
  if (d_stream) {
    EmitParams ep{d_frames, d_halo, jp.nframes, jp.npix, jp.H, jp.W, jp.px, jp.py, d_sel, d_stream,
                  0, jp.npix};
    CUDA_TRY(launch_emit_any(ep, st));
    ++launches;
  }
  g_launches = launches;
  if (g_profile) {
    cudaEventRecord(tc.e2, st);
    tc.launches = launches;
    g_timed.push_back(tc);
  }
  return PCBZ_OK;
}

int check_err_flag(const Plan &pl, void *d_ws, cudaStream_t st) {
  int flag = 0;
  CUDA_TRY(cudaMemcpyAsync(&flag, static_cast<char *>(d_ws) + pl.off_err, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (flag) return fail(PCBZ_E_INTERNAL, "judge kernel reported internal error %d", flag);
  return PCBZ_OK;
}

}  // namespace

extern "C" {

const char *pcbz_version(void) { return "pcbz_b200 0.1.0 sm_100a"; }

// ---- host memory helpers of the whole-compressor path ---------------------
// Page-locked host memory: device->host copies into it run at PCIe speed
// (pageable destinations measured 4.8 GB/s for the 573 MB of C2 payloads).
void *pcbz_host_alloc(size_t bytes) {
  void *p = nullptr;
  if (cudaHostAlloc(&p, std::max<size_t>(bytes, 1), cudaHostAllocDefault) != cudaSuccess) {
    fail(PCBZ_E_CUDA, "cudaHostAlloc of %zu bytes failed", bytes);
    return nullptr;
  }
  return p;
}

int pcbz_host_free(void *p) {
  if (p) CUDA_TRY(cudaFreeHost(p));
  return PCBZ_OK;
}

// dst = src[0][:len[0]] ++ src[1][:len[1]] ++ ..., copied by up to `threads`
// host threads over equal byte ranges (a fresh destination is first-touched
// in parallel, which is what bounds a single-threaded join).
int pcbz_gather(uint8_t *dst, const uint8_t *const *src, const int64_t *len, int64_t n, int threads) {
  if (n < 0 || (n > 0 && (!dst || !src || !len))) return fail(PCBZ_E_INVALID, "invalid gather arguments");
  std::vector<int64_t> off(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) {
    if (len[i] < 0 || (len[i] > 0 && !src[i])) return fail(PCBZ_E_INVALID, "invalid piece %lld", (long long)i);
    off[i + 1] = off[i] + len[i];
  }
  const int64_t total = off[n];
  const int64_t nt = std::max<int64_t>(1, std::min<int64_t>({(int64_t)std::max(threads, 1), total >> 22, 64}));
  auto work = [&](int64_t t) {
    const int64_t a = total * t / nt, b = total * (t + 1) / nt;
    int64_t i = std::upper_bound(off.begin(), off.end(), a) - off.begin() - 1;
    for (int64_t x = a; x < b && i < n; ++i) {
      const int64_t lo = std::max(x, off[i]), hi = std::min(b, off[i + 1]);
      if (hi > lo) memcpy(dst + lo, src[i] + (lo - off[i]), (size_t)(hi - lo));
      x = hi;
    }
  };
  std::vector<std::thread> pool;
  for (int64_t t = 1; t < nt; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto &th : pool) th.join();
  return PCBZ_OK;
}

const char *pcbz_last_error(void) { return g_err.c_str(); }

int pcbz_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  int good = 0;
  for (int d = 0; d < n; ++d) {
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d);
    good += major == 10;
  }
  return good;
}

int pcbz_set_profiling(int on) {
  g_profile = on != 0;
  return PCBZ_OK;
}

int pcbz_last_timing(float *hist_ms, float *total_ms, int *launches) {
  float hs = 0.f, ts = 0.f;
  int nl = 0;
  for (TimedCall &tc : g_timed) {
    float a = 0.f, b = 0.f;
    CUDA_TRY(cudaEventSynchronize(tc.e2));
    CUDA_TRY(cudaEventElapsedTime(&a, tc.e0, tc.e1));
    CUDA_TRY(cudaEventElapsedTime(&b, tc.e0, tc.e2));
    hs += a; ts += b; nl += tc.launches;
    cudaEventDestroy(tc.e0); cudaEventDestroy(tc.e1); cudaEventDestroy(tc.e2);
  }
  const bool any = !g_timed.empty();
  g_timed.clear();
  if (hist_ms) *hist_ms = hs;
  if (total_ms) *total_ms = ts;
  if (launches) *launches = any ? nl : g_launches;
  return PCBZ_OK;
}

size_t pcbz_judge_workspace_size(int64_t nframes, int64_t h, int64_t w, int k, int want_hist) {
  if (nframes < 1 || h < 1 || w < 1 || k < 1 || k > PCBZ_MAX_CANDIDATES) return 0;
  return workspace_upper_bound(nframes, h, w, k, want_hist != 0, 1);
}

int pcbz_judge_device(const uint16_t *d_frames, const uint16_t *d_halo_prev, int64_t nframes,
                      int64_t h, int64_t w, int64_t px, int64_t py, const uint8_t *specs, int k,
                      int temporal, double *d_ent_out, uint8_t *d_sel_out, uint8_t *d_stream_out,
                      uint32_t *d_hist_out, void *d_workspace, size_t workspace_bytes,
                      void *stream) {
  int rc = check_device();
  if (rc) return rc;
  Plan pl;
  rc = make_plan(nframes, h, w, px, py, specs, k, d_halo_prev != nullptr, temporal,
                 d_hist_out != nullptr, pl);
  if (rc) return rc;
  if (workspace_bytes < pl.ws_bytes)
    return fail(PCBZ_E_INVALID, "workspace too small: %zu < %zu bytes", workspace_bytes, pl.ws_bytes);
  return run_plan(pl, d_frames, d_halo_prev, d_ent_out, d_sel_out, d_stream_out, d_hist_out,
                  d_workspace, static_cast<cudaStream_t>(stream));
}

// Frame counts of the pipeline chunks of pcbz_judge_host: uploads of chunk
// i+1, the judge of chunk i and downloads of chunk i-1 overlap, so the first
// upload and the last download are exposed.  A chunk holds ~135 items
// (frames x candidates x segments of the call's plan, about one wave of the
// persistent grid): C2 (13 items / frame) 10 frames, C3 (26) 5, C4 (26 x 8
// segments) 1 -- measured e2e, frames per chunk: C2 9 / 10 / 11 / 12 ->
// 39.0 / 39.1 / 38.0 / 37.7 GB/s; C3 4 / 5 / 6 / 7 / 10 -> 22.0 / 23.1 /
// 23.4 / 23.1 / 22.5; C4 1 / 2 / 3 / 4 / 8 -> 22.0 / 19.5 / 17.9 / 15.6 /
// 13.3 (profiles/r02_notes.md).  Volumes under 128 MB (PCBZ_HOST_BIG_MB)
// stay one chunk.  Optional ramps (PCBZ_HOST_RAMP / PCBZ_HOST_RAMP_DOWN: doubling
// from that many frames at the start / halving to it at the end) shorten the
// exposed ends; PCBZ_HOST_CHUNK forces the base size.
std::vector<int64_t> host_chunks(int64_t nframes, int64_t frame_bytes, int64_t items_per_frame) {
  auto env = [](const char *name) -> int64_t {
    const char *e = getenv(name);
    return e ? atoll(e) : 0;
  };
  static const int64_t forced = env("PCBZ_HOST_CHUNK");
  static const int64_t ramp = env("PCBZ_HOST_RAMP");            // first chunk size of the ramp-up
  static const int64_t ramp_down = env("PCBZ_HOST_RAMP_DOWN");  // last chunk size of the ramp-down
  static const int64_t big = [] {   // PCBZ_HOST_BIG_MB: volume size that pipelines < 16 frames
    const char *e = getenv("PCBZ_HOST_BIG_MB");
    return (int64_t)(e ? atoll(e) : 128) << 20;
  }();
  if (forced <= 0 && (nframes < 2 || nframes * frame_bytes < big))
    return {nframes};  // too little to pay for a pipeline
  const int64_t per_chunk = (135 + std::max<int64_t>(items_per_frame, 1) / 2) / std::max<int64_t>(items_per_frame, 1);
  const int64_t base = std::min(nframes, forced > 0 ? forced : std::max<int64_t>(1, per_chunk));
  std::vector<int64_t> head, tail, out;
  int64_t left = nframes;
  for (int64_t c = ramp; c > 0 && c < base && left >= 4 * c; c *= 2) {
    head.push_back(c);
    left -= c;
  }
  for (int64_t c = ramp_down; c > 0 && c < base && left >= 4 * c; c *= 2) {
    tail.push_back(c);
    left -= c;
  }
  out = head;
  while (left > 0) {
    const int64_t c = std::min(base, left);
    out.push_back(c);
    left -= c;
  }
  out.insert(out.end(), tail.rbegin(), tail.rend());
  return out;
}

int pcbz_judge_host(const uint16_t *frames, const uint16_t *halo_prev, int64_t nframes, int64_t h,
                    int64_t w, int64_t px, int64_t py, const uint8_t *specs, int k, int temporal,
                    double *ent_out, uint8_t *sel_out, uint8_t *stream_out) {
  HostCtx &c = g_ctx;
  int rc = c.init();
  if (rc) return rc;
  Plan full;  // validates the whole call up front
  rc = make_plan(nframes, h, w, px, py, specs, k, halo_prev != nullptr, temporal, false, full);
  if (rc) return rc;
  const int64_t npix = h * w;
  const size_t fbytes = (size_t)nframes * npix * 2;
  const std::vector<int64_t> sizes = host_chunks(nframes, npix * 2, (int64_t)k * full.jp.S);
  const int64_t nchunks = (int64_t)sizes.size();
  std::vector<int64_t> starts(nchunks + 1, 0);
  for (int64_t i = 0; i < nchunks; ++i) starts[i + 1] = starts[i] + sizes[i];
  // Chunks alternate between two compute streams (one workspace each), so the
  // last, partly filled wave of chunk i overlaps the start of chunk i+1; the
  // segment count is planned for the whole call's pairs accordingly.
  // The first `head` / last `tail` chunks choose their segment count for
  // their own pairs (shorter items: the GPU fills before many frames have
  // arrived, and the final judge -- and the download behind it -- finishes
  // sooner); the others plan for the whole call (PCBZ_HOST_HEAD / _TAIL).
  static const int64_t tail = [] {
    const char *e = getenv("PCBZ_HOST_TAIL");
    return (int64_t)(e ? atoll(e) : 0);
  }();
  static const int64_t head = [] {
    const char *e = getenv("PCBZ_HOST_HEAD");
    return (int64_t)(e ? atoll(e) : 0);
  }();
  static const int edge_s = [] {   // segment count of the head / tail chunks (0: their own plan)
    const char *e = getenv("PCBZ_HOST_EDGE_S");
    return e ? atoi(e) : 0;
  }();
  auto chunk_plan = [&](int64_t i, Plan &pl) {
    const int64_t a = starts[i], n = sizes[i];
    const bool own = i >= nchunks - tail || i < head;
    const int saved = g_seg_override;
    if (own && edge_s > 0) g_seg_override = edge_s;
    const int r = make_plan(n, h, w, px, py, specs, k, a > 0 ? temporal != 0 : halo_prev != nullptr,
                            temporal, false, pl, 1, 0, own ? 0 : full.jp.npairs);
    g_seg_override = saved;
    return r;
  };
  size_t ws_bytes = 0;
  for (int64_t i = 0; i < nchunks; ++i) {
    Plan pl;
    if ((rc = chunk_plan(i, pl))) return rc;
    ws_bytes = std::max(ws_bytes, pl.ws_bytes);
  }
  ws_bytes = align_up(ws_bytes);
  // compute streams (one workspace each) that chunks rotate over
  static const int nstreams = [] {
    const char *e = getenv("PCBZ_HOST_STREAMS");
    const int v = e ? atoi(e) : 2;
    return v < 1 ? 1 : (v > 32 ? 32 : v);
  }();
  const int nws = (int)std::min<int64_t>(nchunks, nstreams);
  if ((rc = c.frames.ensure(fbytes)) || (rc = c.ent.ensure((size_t)nframes * k * 8)) ||
      (rc = c.sel.ensure((size_t)nframes)) || (rc = c.ws.ensure(nws * ws_bytes + 256)))
    return rc;
  if (halo_prev && (rc = c.prev.ensure((size_t)npix * 2))) return rc;
  if (stream_out && (rc = c.stream_out.ensure(fbytes))) return rc;
  if (!c.s_in) {
    CUDA_TRY(cudaStreamCreateWithFlags(&c.s_in, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&c.s_out, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&c.s_comp2, cudaStreamNonBlocking));
  }
  while ((int)c.s_more.size() + 2 < nws) {
    cudaStream_t x;
    CUDA_TRY(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    c.s_more.push_back(x);
  }
  std::vector<cudaStream_t> comp = {c.stream, c.s_comp2};
  for (cudaStream_t x : c.s_more) comp.push_back(x);
  comp.resize(std::max(nws, 1));
  int *d_err = reinterpret_cast<int *>(c.ws.as<char>() + nws * ws_bytes);  // shared by all chunks
  std::vector<cudaEvent_t> ev(2 * nchunks + 1);
  for (auto &e : ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  // every compute stream starts after the error word is cleared
  CUDA_TRY(cudaMemsetAsync(d_err, 0, 4, comp[0]));
  CUDA_TRY(cudaEventRecord(ev[2 * nchunks], comp[0]));
  for (int q = 1; q < nws; ++q) CUDA_TRY(cudaStreamWaitEvent(comp[q], ev[2 * nchunks], 0));
  if (halo_prev)
    CUDA_TRY(cudaMemcpyAsync(c.prev.p, halo_prev, (size_t)npix * 2, cudaMemcpyHostToDevice, c.s_in));
  const uint16_t *d_frames = c.frames.as<uint16_t>();
  // PCBZ_HOST_TRACE=1: per-chunk timeline (upload end, judge end, download
  // end, ms after the call's first upload) on stderr, for tuning the chunks
  static const bool trace = getenv("PCBZ_HOST_TRACE") != nullptr;
  std::vector<cudaEvent_t> tev;
  if (trace) {
    tev.resize(3 * nchunks + 1);
    for (auto &e : tev) CUDA_TRY(cudaEventCreate(&e));
    CUDA_TRY(cudaEventRecord(tev[3 * nchunks], c.s_in));
  }
  for (int64_t i = 0; i < nchunks; ++i) {
    const int64_t a = starts[i], n = sizes[i];
    const size_t off = (size_t)a * npix;
    cudaStream_t st = comp[i % nws];
    char *ws = c.ws.as<char>() + (i % nws) * ws_bytes;
    CUDA_TRY(cudaMemcpyAsync(c.frames.as<uint16_t>() + off, frames + off, (size_t)n * npix * 2,
                             cudaMemcpyHostToDevice, c.s_in));
    CUDA_TRY(cudaEventRecord(ev[2 * i], c.s_in));
    if (trace) CUDA_TRY(cudaEventRecord(tev[3 * i], c.s_in));
    CUDA_TRY(cudaStreamWaitEvent(st, ev[2 * i], 0));
    // the previous frame of chunk i's first frame: the halo (chunk 0) or frame
    // a-1, uploaded earlier on the same (in-order) copy stream
    const uint16_t *d_halo = a > 0 ? (temporal ? d_frames + off - npix : nullptr)
                                   : (halo_prev ? c.prev.as<uint16_t>() : nullptr);
    Plan pl;
    if ((rc = chunk_plan(i, pl))) return rc;
    rc = run_plan(pl, d_frames + off, d_halo, c.ent.as<double>() + a * k, c.sel.as<uint8_t>() + a,
                  stream_out ? c.stream_out.as<uint8_t>() + 2 * off : nullptr, nullptr, ws, st, d_err);
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(ev[2 * i + 1], st));
    if (trace) CUDA_TRY(cudaEventRecord(tev[3 * i + 1], st));
    CUDA_TRY(cudaStreamWaitEvent(c.s_out, ev[2 * i + 1], 0));
    CUDA_TRY(cudaMemcpyAsync(ent_out + a * k, c.ent.as<double>() + a * k, (size_t)n * k * 8,
                             cudaMemcpyDeviceToHost, c.s_out));
    CUDA_TRY(cudaMemcpyAsync(sel_out + a, c.sel.as<uint8_t>() + a, (size_t)n, cudaMemcpyDeviceToHost,
                             c.s_out));
    if (stream_out)
      CUDA_TRY(cudaMemcpyAsync(stream_out + 2 * off, c.stream_out.as<uint8_t>() + 2 * off,
                               (size_t)n * npix * 2, cudaMemcpyDeviceToHost, c.s_out));
    if (trace) CUDA_TRY(cudaEventRecord(tev[3 * i + 2], c.s_out));
  }
  int flag = 0;
  CUDA_TRY(cudaStreamSynchronize(c.s_out));  // every chunk's judge precedes its D2H
  if (trace) {
    for (int64_t i = 0; i < nchunks; ++i) {
      float t[3];
      for (int j = 0; j < 3; ++j) CUDA_TRY(cudaEventElapsedTime(&t[j], tev[3 * nchunks], tev[3 * i + j]));
      fprintf(stderr, "pcbz_judge_host chunk %lld (%lld frames): up %.3f judged %.3f down %.3f ms\n",
              (long long)i, (long long)sizes[i], t[0], t[1], t[2]);
    }
    for (auto &e : tev) cudaEventDestroy(e);
  }
  CUDA_TRY(cudaMemcpy(&flag, d_err, 4, cudaMemcpyDeviceToHost));
  for (auto &e : ev) cudaEventDestroy(e);
  if (flag) return fail(PCBZ_E_INTERNAL, "judge kernel reported internal error %d", flag);
  return PCBZ_OK;
}

int pcbz_select_predictor(const uint16_t *frame, const uint16_t *prev, int64_t h, int64_t w,
                          int64_t px, int64_t py, const uint8_t *specs, int k, double *ent_out,
                          uint8_t *selected, int64_t *hist_out) {
  bool any_temporal = false;
  for (int i = 0; i < k; ++i) any_temporal |= (specs[i] & 0x80) != 0;
  if (any_temporal && !prev) return fail(PCBZ_E_INVALID, "temporal candidate given but no previous frame");
  HostCtx &c = g_ctx;
  int rc = c.init();
  if (rc) return rc;
  // the previous frame rides as the "halo" of a one-frame sequence, so every
  // candidate (temporal ones included) is scored on frame 0 only
  const int64_t nfr = 1;
  Plan pl;
  rc = make_plan(nfr, h, w, px, py, specs, k, prev != nullptr, 1, hist_out != nullptr, pl);
  if (rc) return rc;
  const size_t fb = (size_t)h * w * 2;
  if ((rc = c.frames.ensure(fb)) || (rc = c.ent.ensure((size_t)k * 8)) ||
      (rc = c.sel.ensure(1)) || (rc = c.ws.ensure(pl.ws_bytes)))
    return rc;
  if (prev && (rc = c.prev.ensure(fb))) return rc;
  if (hist_out && (rc = c.hist.ensure((size_t)k * 65536 * 4))) return rc;
  cudaStream_t st = c.stream;
  if (prev) CUDA_TRY(cudaMemcpyAsync(c.prev.p, prev, fb, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(c.frames.p, frame, fb, cudaMemcpyHostToDevice, st));
  rc = run_plan(pl, c.frames.as<uint16_t>(), prev ? c.prev.as<uint16_t>() : nullptr,
                c.ent.as<double>(), c.sel.as<uint8_t>(), nullptr,
                hist_out ? c.hist.as<uint32_t>() : nullptr, c.ws.p, st);
  if (rc) return rc;
  std::vector<double> ent((size_t)nfr * k);
  std::vector<uint8_t> sel(nfr);
  CUDA_TRY(cudaMemcpyAsync(ent.data(), c.ent.p, ent.size() * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(sel.data(), c.sel.p, nfr, cudaMemcpyDeviceToHost, st));
  std::vector<uint32_t> h32;
  if (hist_out) {
    h32.resize((size_t)k * 65536);
    CUDA_TRY(cudaMemcpyAsync(h32.data(), c.hist.as<uint32_t>() + (size_t)(nfr - 1) * k * 65536,
                             h32.size() * 4, cudaMemcpyDeviceToHost, st));
  }
  rc = check_err_flag(pl, c.ws.p, st);
  if (rc) return rc;
  memcpy(ent_out, ent.data() + (size_t)(nfr - 1) * k, (size_t)k * 8);
  *selected = sel[nfr - 1];
  if (hist_out)
    for (size_t i = 0; i < h32.size(); ++i) hist_out[i] = h32[i];
  return PCBZ_OK;
}

int pcbz_residual_bwt_pair_hist(const uint16_t *img, int64_t h, int64_t w, int intra_id,
                                int64_t px, int64_t py, int64_t *hist_out) {
  if (intra_id < 0 || intra_id > 12) return fail(PCBZ_E_INVALID, "intra predictor id must be in [0, 12], got %d", intra_id);
  const uint8_t spec = (uint8_t)intra_id;
  double ent = 0;
  uint8_t sel = 0;
  return pcbz_select_predictor(img, nullptr, h, w, px, py, &spec, 1, &ent, &sel, hist_out);
}

int pcbz_residual_image(const uint16_t *img, int64_t h, int64_t w, int intra_id, int64_t px,
                        int64_t py, uint16_t *out) {
  int rc = validate_geometry(h, w, px, py);
  if (rc) return rc;
  if (intra_id < 0 || intra_id > 12) return fail(PCBZ_E_INVALID, "intra predictor id must be in [0, 12], got %d", intra_id);
  HostCtx &c = g_ctx;
  if ((rc = c.init())) return rc;
  const size_t nb = (size_t)h * w * 2;
  if ((rc = c.frames.ensure(nb)) || (rc = c.out.ensure(nb))) return rc;
  cudaStream_t st = c.stream;
  CUDA_TRY(cudaMemcpyAsync(c.frames.p, img, nb, cudaMemcpyHostToDevice, st));
  CUDA_TRY(launch_residual_image(c.frames.as<uint16_t>(), nullptr, h, w, intra_id, (int)px, (int)py,
                                 c.out.as<uint16_t>(), 0, st));
  CUDA_TRY(cudaMemcpyAsync(out, c.out.p, nb, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return PCBZ_OK;
}

int pcbz_temporal_delta(const uint16_t *cur, const uint16_t *prev, int64_t n, uint16_t *out) {
  if (n < 0) return fail(PCBZ_E_INVALID, "negative length");
  if (n == 0) return PCBZ_OK;
  HostCtx &c = g_ctx;
  int rc = c.init();
  if (rc) return rc;
  const size_t nb = (size_t)n * 2;
  if ((rc = c.frames.ensure(nb)) || (rc = c.prev.ensure(nb)) || (rc = c.out.ensure(nb))) return rc;
  cudaStream_t st = c.stream;
  CUDA_TRY(cudaMemcpyAsync(c.frames.p, cur, nb, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(c.prev.p, prev, nb, cudaMemcpyHostToDevice, st));
  CUDA_TRY(launch_temporal_delta(c.frames.as<uint16_t>(), c.prev.as<uint16_t>(), n, c.out.as<uint16_t>(), st));
  CUDA_TRY(cudaMemcpyAsync(out, c.out.p, nb, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return PCBZ_OK;
}

int pcbz_counting_bwt(const uint8_t *s, int64_t n, uint8_t *out) {
  if (n < 0) return fail(PCBZ_E_INVALID, "negative length");
  if (n == 0) return PCBZ_OK;
  HostCtx &c = g_ctx;
  int rc = c.init();
  if (rc) return rc;
  const size_t sw = counting_bwt_scratch_words(n);
  if ((rc = c.bytes.ensure((size_t)n)) || (rc = c.out.ensure((size_t)n)) || (rc = c.scratch.ensure(sw * 4))) return rc;
  cudaStream_t st = c.stream;
  CUDA_TRY(cudaMemcpyAsync(c.bytes.p, s, (size_t)n, cudaMemcpyHostToDevice, st));
  CUDA_TRY(launch_counting_bwt(c.bytes.as<uint8_t>(), n, c.out.as<uint8_t>(), c.scratch.as<uint32_t>(), sw, st));
  CUDA_TRY(cudaMemcpyAsync(out, c.out.p, (size_t)n, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return PCBZ_OK;
}

static int pair_hist_dev(HostCtx &c, const uint8_t *d_s, int64_t n, int64_t *hist_out) {
  int rc = c.hist.ensure(65536 * 4);
  if (rc) return rc;
  cudaStream_t st = c.stream;
  CUDA_TRY(cudaMemsetAsync(c.hist.p, 0, 65536 * 4, st));
  if (n >= 2) CUDA_TRY(launch_pair_hist(d_s, n, c.hist.as<uint32_t>(), st));
  std::vector<uint32_t> h32(65536);
  CUDA_TRY(cudaMemcpyAsync(h32.data(), c.hist.p, 65536 * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  for (int i = 0; i < 65536; ++i) hist_out[i] = h32[i];
  return PCBZ_OK;
}

int pcbz_pair_hist(const uint8_t *s, int64_t n, int64_t *hist_out) {
  if (n < 0) return fail(PCBZ_E_INVALID, "negative length");
  HostCtx &c = g_ctx;
  int rc = c.init();
  if (rc) return rc;
  if ((rc = c.bytes.ensure((size_t)std::max<int64_t>(n, 1)))) return rc;
  if (n) CUDA_TRY(cudaMemcpyAsync(c.bytes.p, s, (size_t)n, cudaMemcpyHostToDevice, c.stream));
  return pair_hist_dev(c, c.bytes.as<uint8_t>(), n, hist_out);
}

int pcbz_bwt_pair_hist(const uint8_t *s, int64_t n, int64_t *hist_out) {
  if (n < 0) return fail(PCBZ_E_INVALID, "negative length");
  HostCtx &c = g_ctx;
  int rc = c.init();
  if (rc) return rc;
  if (n < 2) {
    for (int i = 0; i < 65536; ++i) hist_out[i] = 0;
    return PCBZ_OK;
  }
  const size_t sw = counting_bwt_scratch_words(n);
  if ((rc = c.bytes.ensure((size_t)n)) || (rc = c.out.ensure((size_t)n)) || (rc = c.scratch.ensure(sw * 4))) return rc;
  cudaStream_t st = c.stream;
  CUDA_TRY(cudaMemcpyAsync(c.bytes.p, s, (size_t)n, cudaMemcpyHostToDevice, st));
  CUDA_TRY(launch_counting_bwt(c.bytes.as<uint8_t>(), n, c.out.as<uint8_t>(), c.scratch.as<uint32_t>(), sw, st));
  return pair_hist_dev(c, c.out.as<uint8_t>(), n, hist_out);
}

int pcbz_entropy2d(const int64_t *counts, int64_t total, double *out) {
  HostCtx &c = g_ctx;
  int rc = c.init();
  if (rc) return rc;
  if ((rc = c.hist.ensure(65536 * 8)) || (rc = c.ent.ensure(8))) return rc;
  cudaStream_t st = c.stream;
  CUDA_TRY(cudaMemcpyAsync(c.hist.p, counts, 65536 * 8, cudaMemcpyHostToDevice, st));
  int64_t nt = 0;
  const double *terms = total > 0 ? registered_terms(total, &nt) : nullptr;
  CUDA_TRY(launch_entropy_u64(c.hist.as<uint64_t>(), total > 0 ? (double)total : 0.0, terms, nt,
                              c.ent.as<double>(), st));
  CUDA_TRY(cudaMemcpyAsync(out, c.ent.p, 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return PCBZ_OK;
}

}  // extern "C"

extern "C" {

// Entropy terms evaluated by the host (e.g. the reference's own numpy):
// terms[c] = p * log2(p) with p = c / total for c = 1..total (terms[0] is
// unused).  Every later judge / entropy call on this device whose total
// matches reduces these exact values (entropy.cuh), so the entropies are
// bit-identical to the host's entropy2d.
int pcbz_register_entropy_terms(int64_t total, const double *terms, int64_t n) {
  if (total < 1 || n != total + 1 || !terms)
    return fail(PCBZ_E_INVALID, "entropy term table needs total >= 1 and total + 1 entries (total=%lld n=%lld)",
                (long long)total, (long long)n);
  int rc = check_device();
  if (rc) return rc;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_terms_mu);
  for (const TermTable &t : g_terms)
    if (t.dev == dev && t.total == total) return PCBZ_OK;
  const size_t bytes = (size_t)n * sizeof(double);
  if (g_terms_bytes + bytes > terms_budget())
    return fail(PCBZ_E_INVALID, "entropy term tables would exceed PCBZ_TERMS_BUDGET_MB (%zu + %zu bytes)",
                g_terms_bytes, bytes);
  double *d = nullptr;
  CUDA_TRY(cudaMalloc(&d, bytes));
  // a pageable cudaMemcpy may return before its DMA lands, and the kernels
  // that read the table run on non-blocking streams: wait for the device
  if (cudaMemcpy(d, terms, bytes, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess) {
    cudaFree(d);
    return fail(PCBZ_E_CUDA, "copy of the entropy term table failed");
  }
  g_terms.push_back({dev, total, d});
  g_terms_bytes += bytes;
  return PCBZ_OK;
}

int pcbz_entropy_terms_registered(int64_t total) {
  int64_t nt = 0;
  return registered_terms(total, &nt) != nullptr ? 1 : 0;
}

int pcbz_set_segment_override(int segments) {
  g_seg_override = segments > 0 ? segments : 0;
  return PCBZ_OK;
}

static int check_sel(const uint8_t *sel, int64_t nframes, bool halo) {
  for (int64_t f = 0; f < nframes; ++f) {
    if ((sel[f] & 0x7F) > 12) return fail(PCBZ_E_INVALID, "invalid intra predictor id %d in byte 0x%02X", sel[f] & 0x7F, sel[f]);
    if (f == 0 && !halo && (sel[f] & 0x80)) return fail(PCBZ_E_INVALID, "temporal predictor requires a previous frame");
  }
  return PCBZ_OK;
}

int pcbz_emit_host(const uint16_t *frames, const uint16_t *halo_prev, int64_t nframes, int64_t h,
                   int64_t w, int64_t px, int64_t py, const uint8_t *sel, uint8_t *stream_out) {
  int rc = validate_geometry(h, w, px, py);
  if (rc) return rc;
  if (nframes < 1) return fail(PCBZ_E_INVALID, "at least one frame is required");
  if ((rc = check_sel(sel, nframes, halo_prev != nullptr))) return rc;
  HostCtx &c = g_ctx;
  if ((rc = c.init())) return rc;
  const size_t fb = (size_t)nframes * h * w * 2;
  if ((rc = c.frames.ensure(fb)) || (rc = c.stream_out.ensure(fb)) || (rc = c.sel.ensure(nframes))) return rc;
  if (halo_prev && (rc = c.prev.ensure((size_t)h * w * 2))) return rc;
  cudaStream_t st = c.stream;
  CUDA_TRY(cudaMemcpyAsync(c.frames.p, frames, fb, cudaMemcpyHostToDevice, st));
  if (halo_prev) CUDA_TRY(cudaMemcpyAsync(c.prev.p, halo_prev, (size_t)h * w * 2, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(c.sel.p, sel, (size_t)nframes, cudaMemcpyHostToDevice, st));
  EmitParams ep{c.frames.as<uint16_t>(), halo_prev ? c.prev.as<uint16_t>() : nullptr, nframes,
                h * w, (int)h, (int)w, (int)px, (int)py, c.sel.as<uint8_t>(), c.stream_out.as<uint8_t>(),
                0, h * w};
  CUDA_TRY(launch_emit_any(ep, st));
  CUDA_TRY(cudaMemcpyAsync(stream_out, c.stream_out.p, fb, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return PCBZ_OK;
}

int pcbz_reconstruct_host(const uint16_t *residuals, const uint16_t *halo_prev, int64_t nframes,
                          int64_t h, int64_t w, int64_t px, int64_t py, const uint8_t *sel,
                          uint16_t *frames_out) {
  int rc = validate_geometry(h, w, px, py);
  if (rc) return rc;
  if (nframes < 1) return fail(PCBZ_E_INVALID, "at least one frame is required");
  if ((rc = check_sel(sel, nframes, halo_prev != nullptr))) return rc;
  HostCtx &c = g_ctx;
  if ((rc = c.init())) return rc;
  const size_t fb = (size_t)nframes * h * w * 2;
  if ((rc = c.frames.ensure(fb)) || (rc = c.out.ensure(fb)) || (rc = c.sel.ensure(nframes))) return rc;
  if (halo_prev && (rc = c.prev.ensure((size_t)h * w * 2))) return rc;
  cudaStream_t st = c.stream;
  CUDA_TRY(cudaMemcpyAsync(c.frames.p, residuals, fb, cudaMemcpyHostToDevice, st));
  if (halo_prev) CUDA_TRY(cudaMemcpyAsync(c.prev.p, halo_prev, (size_t)h * w * 2, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(c.sel.p, sel, (size_t)nframes, cudaMemcpyHostToDevice, st));
  CUDA_TRY(launch_reconstruct(c.frames.as<uint16_t>(), halo_prev ? c.prev.as<uint16_t>() : nullptr,
                              nframes, h, w, (int)px, (int)py, c.sel.as<uint8_t>(), c.out.as<uint16_t>(), st));
  CUDA_TRY(cudaMemcpyAsync(frames_out, c.out.p, fb, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return PCBZ_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// band sharding: every stream cut into nbands contiguous pixel bands (one per
// rank); partial histograms + segment summaries are combined by the caller's
// collective (sum / gather) and finished by pcbz_judge_merge_device
// ---------------------------------------------------------------------------

extern "C" {

int pcbz_band_layout(int64_t nframes, int64_t h, int64_t w, int64_t px, int64_t py,
                     const uint8_t *specs, int k, int temporal, int has_halo, int nbands,
                     int *segments_per_band, size_t *summary_bytes, size_t *workspace_bytes) {
  Plan pl;
  int rc = make_plan(nframes, h, w, px, py, specs, k, has_halo != 0, temporal, true, pl, nbands, 0);
  if (rc) return rc;
  if (segments_per_band) *segments_per_band = pl.jp.S;
  if (summary_bytes) *summary_bytes = (size_t)nframes * k * pl.jp.S * 512 * sizeof(int16_t);
  if (workspace_bytes) *workspace_bytes = pl.ws_bytes;
  return PCBZ_OK;
}

int pcbz_band_range(int64_t h, int64_t w, int nbands, int band, int64_t *pix_begin,
                    int64_t *pix_end) {
  const int64_t npix = h * w;
  if (h < 1 || w < 1 || nbands < 1 || band < 0 || band >= nbands)
    return fail(PCBZ_E_INVALID, "band %d of %d invalid for a %lldx%lld frame", band, nbands,
                (long long)h, (long long)w);
  // 8-pixel granules when possible, so every band emits with the chunk kernel
  const int64_t g = npix % 8 == 0 ? 8 : 1, n = npix / g;
  *pix_begin = g * (n * band / nbands);
  *pix_end = g * (n * (band + 1) / nbands);
  return PCBZ_OK;
}

int pcbz_judge_band_device(const uint16_t *d_frames, const uint16_t *d_halo_prev, int64_t nframes,
                           int64_t h, int64_t w, int64_t px, int64_t py, const uint8_t *specs, int k,
                           int temporal, int band, int nbands, uint32_t *d_hist_out,
                           int16_t *d_summary_out, void *d_workspace, size_t workspace_bytes,
                           void *stream) {
  int rc = check_device();
  if (rc) return rc;
  if (!d_hist_out || !d_summary_out) return fail(PCBZ_E_INVALID, "band judge needs histogram and summary outputs");
  Plan pl;
  rc = make_plan(nframes, h, w, px, py, specs, k, d_halo_prev != nullptr, temporal, true, pl,
                 nbands, band);
  if (rc) return rc;
  if (workspace_bytes < pl.ws_bytes)
    return fail(PCBZ_E_INVALID, "workspace too small: %zu < %zu bytes", workspace_bytes, pl.ws_bytes);
  JudgeParams &jp = pl.jp;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char *ws = static_cast<char *>(d_workspace);
  jp.frames = d_frames;
  jp.halo = d_halo_prev;
  if ((reinterpret_cast<uintptr_t>(d_frames) | reinterpret_cast<uintptr_t>(d_halo_prev)) & 15) jp.fast_px = 0;
  jp.ent = nullptr;
  jp.counter = reinterpret_cast<int *>(ws + pl.off_counter);
  jp.err = reinterpret_cast<int *>(ws + pl.off_err);
  jp.fscratch = reinterpret_cast<uint8_t *>(ws + pl.off_fscratch);
  jp.ghist = d_hist_out;
  jp.part = reinterpret_cast<uint32_t *>(ws + pl.off_part);
  // the kernel writes band 0's slot of the summary array: point it at this band
  jp.segsum = d_summary_out - (size_t)band * jp.nslots * jp.S * 512;
  TimedCall tc{nullptr, nullptr, nullptr, 1};
  if (g_profile) {
    cudaEventCreate(&tc.e0); cudaEventCreate(&tc.e1); cudaEventCreate(&tc.e2);
    cudaEventRecord(tc.e0, st);
  }
  CUDA_TRY(cudaMemsetAsync(ws, 0, pl.off_fscratch, st));
  // temporal candidates on materialised delta frames (whole frames: rows
  // outside this band's neighbourhood may hold anything and are never read)
  uint16_t *d_delta = nullptr;
  jp.delta = nullptr;
  const int64_t delta_f0 = d_halo_prev ? 0 : 1;
  int launches = 2;
  if (use_delta(jp, d_frames, d_halo_prev, true) && jp.nframes > delta_f0) {
    CUDA_TRY(pooled_alloc(reinterpret_cast<void **>(&d_delta), (size_t)jp.nframes * jp.npix * 2, st));
    // only the rows this band reads: its own, py + 1 above, and for band 0
    // the last py + 1 rows (the wrapped predecessor of stream byte 0)
    int64_t b0 = 0, b1 = 0;
    if ((rc = pcbz_band_range(h, w, nbands, band, &b0, &b1))) return rc;
    const int64_t above = (py + 1) * w;
    const int64_t r0 = std::max<int64_t>(0, (b0 / w) * w - above) & ~7ll;
    const int64_t r1 = std::min<int64_t>(jp.npix, ((b1 + w - 1) / w * w + 7) & ~7ll);
    CUDA_TRY(launch_delta_frames(d_frames, d_halo_prev, jp.nframes, jp.npix, delta_f0, r0, r1, d_delta, st));
    if (band == 0) {
      const int64_t t0 = std::max<int64_t>(r1, jp.npix - above);
      CUDA_TRY(launch_delta_frames(d_frames, d_halo_prev, jp.nframes, jp.npix, delta_f0, t0 & ~7ll, jp.npix,
                                   d_delta, st));
    }
    jp.delta = d_delta;
    ++launches;
  }
  CUDA_TRY(launch_judge(jp, pl.grid, st));
  if (d_delta) CUDA_TRY(cudaFreeAsync(d_delta, st));
  CUDA_TRY(launch_reduce_parts(jp, st));   // writes every row of d_hist_out
  g_launches = launches;
  if (g_profile) {
    cudaEventRecord(tc.e1, st);
    cudaEventRecord(tc.e2, st);
    g_timed.push_back(tc);
  }
  return PCBZ_OK;
}

int pcbz_judge_merge_device(int64_t nframes, int64_t h, int64_t w, int64_t px, int64_t py,
                            const uint8_t *specs, int k, int temporal, int has_halo, int nbands,
                            uint32_t *d_hist_inout, const int16_t *d_summaries, double *d_ent_out,
                            uint8_t *d_sel_out, void *stream) {
  int rc = check_device();
  if (rc) return rc;
  Plan pl;
  rc = make_plan(nframes, h, w, px, py, specs, k, has_halo != 0, temporal, true, pl, nbands, 0);
  if (rc) return rc;
  JudgeParams &jp = pl.jp;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  jp.ghist = d_hist_inout;
  jp.segsum = const_cast<int16_t *>(d_summaries);
  jp.ent = d_ent_out;
  double *terms = nullptr;  // stream-ordered scratch: this entry point has no workspace
  const bool host_terms = use_registered_terms(jp);
  if (!host_terms) {
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void **>(&terms), kTermTable * sizeof(double), st));
    CUDA_TRY(launch_term_table((double)(2 * jp.npix - 1), terms, st));
    jp.terms = terms;
    jp.nterms = kTermTable;
  }
  CUDA_TRY(cudaMemsetAsync(d_ent_out, 0xFF, (size_t)nframes * k * sizeof(double), st));  // NaN
  CUDA_TRY(launch_finalize(jp, st));
  CUDA_TRY(launch_select(jp, d_sel_out, st));
  if (terms) CUDA_TRY(cudaFreeAsync(terms, st));
  g_launches = host_terms ? 2 : 3;
  return PCBZ_OK;
}

int pcbz_judge_merge_slots_device(int64_t nframes, int64_t h, int64_t w, int64_t px, int64_t py,
                                  const uint8_t *specs, int k, int temporal, int has_halo, int nbands,
                                  int64_t slot_begin, int64_t slot_count, uint32_t *d_hist_owned,
                                  const int16_t *d_summaries_owned, double *d_ent_owned, void *stream) {
  int rc = check_device();
  if (rc) return rc;
  if (slot_begin < 0 || slot_count < 0)
    return fail(PCBZ_E_INVALID, "invalid slot range [%lld, +%lld)", (long long)slot_begin, (long long)slot_count);
  Plan pl;
  rc = make_plan(nframes, h, w, px, py, specs, k, has_halo != 0, temporal, true, pl, nbands, 0);
  if (rc) return rc;
  JudgeParams &jp = pl.jp;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  g_launches = 0;
  if (slot_count == 0) return PCBZ_OK;
  jp.slot0 = slot_begin;
  jp.slot_count = slot_count;
  jp.nslots = slot_count;           // stride of the owned summaries [nbands][slot_count][S][512]
  jp.ghist = d_hist_owned;
  jp.segsum = const_cast<int16_t *>(d_summaries_owned);
  jp.ent = d_ent_owned;
  double *terms = nullptr;
  const bool host_terms = use_registered_terms(jp);
  if (!host_terms) {
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void **>(&terms), kTermTable * sizeof(double), st));
    CUDA_TRY(launch_term_table((double)(2 * jp.npix - 1), terms, st));
    jp.terms = terms;
    jp.nterms = kTermTable;
  }
  CUDA_TRY(cudaMemsetAsync(d_ent_owned, 0xFF, (size_t)slot_count * sizeof(double), st));  // NaN
  CUDA_TRY(launch_finalize_slots(jp, st));
  if (terms) CUDA_TRY(cudaFreeAsync(terms, st));
  g_launches = host_terms ? 1 : 2;
  return PCBZ_OK;
}

int pcbz_judge_merge_peers_device(int64_t nframes, int64_t h, int64_t w, int64_t px, int64_t py,
                                  const uint8_t *specs, int k, int temporal, int has_halo, int nbands,
                                  int band, const uint64_t *d_peer_hist, const uint64_t *d_peer_summaries,
                                  const uint64_t *d_peer_ent, uint32_t *d_hist_scratch, double *d_ent_owned,
                                  void *stream) {
  int rc = check_device();
  if (rc) return rc;
  if (!d_peer_hist || !d_peer_summaries || !d_peer_ent || !d_hist_scratch || !d_ent_owned)
    return fail(PCBZ_E_INVALID, "peer merge needs the peer pointer arrays and the owned buffers");
  if (band < 0 || band >= nbands)
    return fail(PCBZ_E_INVALID, "band %d of %d invalid", band, nbands);
  Plan pl;
  rc = make_plan(nframes, h, w, px, py, specs, k, has_halo != 0, temporal, true, pl, nbands, 0);
  if (rc) return rc;
  JudgeParams &jp = pl.jp;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  g_launches = 0;
  const int64_t q = (nframes * k + nbands - 1) / nbands;   // owned slots per rank (shard.BandBuffers)
  jp.slot0 = (int64_t)band * q;
  jp.slot_count = q;
  jp.nslots = q;
  jp.ghist = d_hist_scratch;
  jp.segsum = nullptr;
  jp.ent = d_ent_owned;
  jp.peer_hist = d_peer_hist;
  jp.peer_summ = d_peer_summaries;
  jp.peer_ent = d_peer_ent;
  double *terms = nullptr;
  const bool host_terms = use_registered_terms(jp);
  if (!host_terms) {
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void **>(&terms), kTermTable * sizeof(double), st));
    CUDA_TRY(launch_term_table((double)(2 * jp.npix - 1), terms, st));
    jp.terms = terms;
    jp.nterms = kTermTable;
  }
  CUDA_TRY(cudaMemsetAsync(d_ent_owned, 0xFF, (size_t)q * sizeof(double), st));  // NaN
  CUDA_TRY(launch_finalize_slots(jp, st));
  if (terms) CUDA_TRY(cudaFreeAsync(terms, st));
  g_launches = host_terms ? 1 : 2;
  return PCBZ_OK;
}

int pcbz_peer_signal(const uint64_t *d_peer_flags, uint32_t *d_my_flags, int nranks, int rank, uint32_t epoch,
                     int mode, void *stream) {
  int rc = check_device();
  if (rc) return rc;
  if (nranks < 1 || rank < 0 || rank >= nranks || mode < 1 || mode > 3)
    return fail(PCBZ_E_INVALID, "peer signal: rank %d of %d, mode %d invalid", rank, nranks, mode);
  if (((mode & 1) && !d_peer_flags) || ((mode & 2) && !d_my_flags))
    return fail(PCBZ_E_INVALID, "peer signal needs the flag arrays");
  CUDA_TRY(launch_peer_signal(d_peer_flags, d_my_flags, nranks, rank, epoch, mode, static_cast<cudaStream_t>(stream)));
  g_launches = 1;
  return PCBZ_OK;
}

int pcbz_judge_select_device(int64_t nframes, const uint8_t *specs, int k, int temporal, int has_halo,
                             const double *d_ent, uint8_t *d_sel_out, void *stream) {
  int rc = check_device();
  if (rc) return rc;
  if (nframes < 1) return fail(PCBZ_E_INVALID, "at least one frame is required");
  if ((rc = validate_specs(specs, k))) return rc;
  JudgeParams jp{};
  if ((rc = build_lists(specs, k, has_halo != 0, temporal, jp.cl))) return rc;
  jp.nframes = nframes;
  jp.ent = const_cast<double *>(d_ent);
  CUDA_TRY(launch_select(jp, d_sel_out, static_cast<cudaStream_t>(stream)));
  g_launches = 1;
  return PCBZ_OK;
}

int pcbz_emit_band_device(const uint16_t *d_frames, const uint16_t *d_halo_prev, int64_t nframes,
                          int64_t h, int64_t w, int64_t px, int64_t py, const uint8_t *d_sel,
                          int band, int nbands, uint8_t *d_stream_out, void *stream) {
  int rc = check_device();
  if (rc) return rc;
  if ((rc = validate_geometry(h, w, px, py))) return rc;
  if (nframes < 1) return fail(PCBZ_E_INVALID, "at least one frame is required");
  int64_t p0 = 0, p1 = 0;
  if ((rc = pcbz_band_range(h, w, nbands, band, &p0, &p1))) return rc;
  g_launches = 0;
  if (p1 == p0) return PCBZ_OK;
  EmitParams ep{d_frames, d_halo_prev, nframes, h * w, (int)h, (int)w, (int)px, (int)py, d_sel,
                d_stream_out, p0, p1};
  CUDA_TRY(launch_emit_any(ep, static_cast<cudaStream_t>(stream)));
  g_launches = 1;
  return PCBZ_OK;
}

}  // extern "C"

extern "C" {

// Testing / tuning hook: while on, every judge call on this thread records
// (smid << 48 | start ns, runs-done ns, end ns) per work item; pcbz_item_trace copies the
// last call's records (item = pair * S + segment) and returns the item count.
int pcbz_set_item_trace(int on) {
  g_trace_on = on != 0;
  return PCBZ_OK;
}

int64_t pcbz_item_trace(uint64_t *out, int64_t max_items, int *segments) {
  if (!g_trace_dev || g_trace_items == 0) return 0;
  const int64_t n = std::min(max_items, g_trace_items);
  if (cudaDeviceSynchronize() != cudaSuccess) return fail(PCBZ_E_CUDA, "trace sync failed");
  if (cudaMemcpy(out, g_trace_dev, (size_t)n * 8 * kTraceWords, cudaMemcpyDeviceToHost) != cudaSuccess)
    return fail(PCBZ_E_CUDA, "trace copy failed");
  if (segments) *segments = g_trace_segments;
  return n;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// judge + emission + bzip2 on the device: pipeline.py:85-108 end to end, only
// the compressed payloads come back
// ---------------------------------------------------------------------------

extern "C" {

size_t pcbz_compress_bound(int64_t nframes, int64_t h, int64_t w, int64_t block_size) {
  if (nframes < 1 || h < 1 || w < 1 || block_size < 1) return 0;
  const int64_t sb = 2 * h * w, nb = (sb + block_size - 1) / block_size;
  size_t b = 0;
  for (int64_t k = 0; k < nb; ++k) b += bz::job_bound(std::min(block_size, sb - k * block_size));
  return b * (size_t)nframes;
}

// frames[f] of a frame-pointer list (no host-side stacking of the volume)
struct FrameSource {
  const uint16_t *base;            // contiguous volume, or
  const uint16_t *const *list;     // one pointer per frame
  int64_t npix;
  const uint16_t *frame(int64_t f) const { return list ? list[f] : base + (size_t)f * npix; }
};

static int compress_impl(const FrameSource &src, const uint16_t *halo_prev, int64_t nframes, int64_t h,
                         int64_t w, int64_t px, int64_t py, const uint8_t *specs, int k, int temporal,
                         const uint8_t *sel_in, int64_t block_size, double *ent_out, uint8_t *sel_out,
                         uint8_t *out, size_t out_cap, int64_t *out_start, int64_t *out_len,
                         uint8_t *raw_flag) {
  static const bool trace = getenv("PCBZ_HOST_TRACE") != nullptr;
  using clk = std::chrono::steady_clock;
  auto ms_since = [](clk::time_point t) {
    return std::chrono::duration<double, std::milli>(clk::now() - t).count();
  };
  int rc = validate_geometry(h, w, px, py);
  if (rc) return rc;
  if (nframes < 1) return fail(PCBZ_E_INVALID, "at least one frame is required");
  if (block_size < 1) return fail(PCBZ_E_INVALID, "block_size must be >= 1, got %lld", (long long)block_size);
  if (sel_in && (rc = check_sel(sel_in, nframes, halo_prev != nullptr))) return rc;
  HostCtx &c = g_ctx;
  if ((rc = c.init())) return rc;
  const int64_t npix = h * w, sb = 2 * npix;
  const int64_t nbf = (sb + block_size - 1) / block_size;     // blocks per frame
  if (out_cap < pcbz_compress_bound(nframes, h, w, block_size))
    return fail(PCBZ_E_INVALID, "output buffer smaller than pcbz_compress_bound");
  // frames per device round: streams of at most 1 GiB (bzip2 batch limit);
  // PCBZ_COMPRESS_ROUND_BYTES lowers it (tests cross round boundaries)
  int64_t round_bytes = (int64_t)1 << 30;
  if (const char *e = getenv("PCBZ_COMPRESS_ROUND_BYTES")) round_bytes = std::min(round_bytes, std::max<int64_t>(1, atoll(e)));
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(nframes, round_bytes / sb));
  cudaStream_t st = c.stream;
  if (halo_prev) {
    if ((rc = c.prev.ensure((size_t)npix * 2))) return rc;
    CUDA_TRY(cudaMemcpyAsync(c.prev.p, halo_prev, (size_t)npix * 2, cudaMemcpyHostToDevice, st));
  }
  size_t used = 0;
  std::vector<int64_t> in_off, o_start, o_len;
  std::vector<uint8_t> host_need;
  for (int64_t a = 0; a < nframes; a += chunk) {
    const int64_t n = std::min(chunk, nframes - a);
    const size_t fb = (size_t)n * npix * 2;
    // the previous frame of this chunk's first frame: halo, or frame a-1
    // (kept in c.prev from the previous round)
    const bool have_prev = a > 0 ? true : halo_prev != nullptr;
    if ((rc = c.frames.ensure(fb)) || (rc = c.stream_out.ensure((size_t)n * sb)) ||
        (rc = c.ent.ensure((size_t)n * std::max(k, 1) * 8)) || (rc = c.sel.ensure((size_t)n)) ||
        (rc = c.out.ensure(pcbz_compress_bound(n, h, w, block_size))))
      return rc;
    if (src.list) {
      for (int64_t f = 0; f < n; ++f)
        CUDA_TRY(cudaMemcpyAsync(c.frames.as<uint16_t>() + (size_t)f * npix, src.frame(a + f), (size_t)npix * 2,
                                 cudaMemcpyHostToDevice, st));
    } else {
      CUDA_TRY(cudaMemcpyAsync(c.frames.p, src.frame(a), fb, cudaMemcpyHostToDevice, st));
    }
    const uint16_t *d_prev = have_prev ? c.prev.as<uint16_t>() : nullptr;
    if (sel_in) {
      CUDA_TRY(cudaMemcpyAsync(c.sel.p, sel_in + a, (size_t)n, cudaMemcpyHostToDevice, st));
      EmitParams ep{c.frames.as<uint16_t>(), d_prev, n, npix, (int)h, (int)w, (int)px, (int)py,
                    c.sel.as<uint8_t>(), c.stream_out.as<uint8_t>(), 0, npix};
      CUDA_TRY(launch_emit_any(ep, st));
    } else {
      Plan pl;
      rc = make_plan(n, h, w, px, py, specs, k, a > 0 ? temporal != 0 : halo_prev != nullptr, temporal, false, pl);
      if (rc) return rc;
      if ((rc = c.ws.ensure(pl.ws_bytes))) return rc;
      rc = run_plan(pl, c.frames.as<uint16_t>(), (a > 0 && temporal) || (a == 0 && halo_prev) ? d_prev : nullptr,
                    c.ent.as<double>(), c.sel.as<uint8_t>(), c.stream_out.as<uint8_t>(), nullptr, c.ws.p, st);
      if (rc) return rc;
      CUDA_TRY(cudaMemcpyAsync(ent_out + a * k, c.ent.p, (size_t)n * k * 8, cudaMemcpyDeviceToHost, st));
      rc = check_err_flag(pl, c.ws.p, st);
      if (rc) return rc;
    }
    CUDA_TRY(cudaMemcpyAsync(sel_out + a, c.sel.p, (size_t)n, cudaMemcpyDeviceToHost, st));
    // the last frame of this round is the next round's previous frame
    if ((rc = c.prev.ensure((size_t)npix * 2))) return rc;
    CUDA_TRY(cudaMemcpyAsync(c.prev.p, c.frames.as<uint16_t>() + (size_t)(n - 1) * npix, (size_t)npix * 2,
                             cudaMemcpyDeviceToDevice, st));
    // bzip2 of every (frame, block) of the round
    const int nj = (int)(n * nbf);
    in_off.assign(nj + 1, 0);
    for (int64_t f = 0; f < n; ++f)
      for (int64_t b = 0; b < nbf; ++b) in_off[f * nbf + b] = f * sb + std::min(b * block_size, sb);
    in_off[nj] = n * sb;
    o_start.assign(nj, 0);
    o_len.assign(nj, 0);
    host_need.assign(nj, 0);
    const size_t cap = pcbz_compress_bound(n, h, w, block_size);
    auto t_round = clk::now();
    if (trace) CUDA_TRY(cudaStreamSynchronize(st));
    const double ms_judge = trace ? ms_since(t_round) : 0.0;
    auto t_bz = clk::now();
    rc = bz::compress_jobs(c.stream_out.as<uint8_t>(), in_off.data(), nj, c.out.as<uint8_t>(), cap,
                           o_start.data(), o_len.data(), host_need.data(), st);
    if (rc) return fail(rc, "%s", bz::last_error());
    const double ms_bz = trace ? ms_since(t_bz) : 0.0;
    auto t_d2h = clk::now();
    size_t coded = 0;
    for (int j = 0; j < nj; ++j) coded = std::max(coded, (size_t)(o_start[j] + o_len[j]));
    if (used + coded > out_cap) return fail(PCBZ_E_INVALID, "output buffer too small");
    if (coded) CUDA_TRY(cudaMemcpy(out + used, c.out.p, coded, cudaMemcpyDeviceToHost));
    for (int j = 0; j < nj; ++j) {
      const size_t g = (size_t)(a * nbf + j);
      raw_flag[g] = host_need[j];
      if (host_need[j]) {  // periodic block: hand the raw bytes to the caller's libbzip2
        const size_t len = (size_t)(in_off[j + 1] - in_off[j]);
        out_start[g] = (int64_t)(used + coded);
        out_len[g] = (int64_t)len;
        if (used + coded + len > out_cap) return fail(PCBZ_E_INVALID, "output buffer too small");
        if (len)
          CUDA_TRY(cudaMemcpy(out + used + coded, c.stream_out.as<uint8_t>() + in_off[j], len, cudaMemcpyDeviceToHost));
        coded += len;
      } else {
        out_start[g] = (int64_t)used + o_start[j];
        out_len[g] = o_len[j];
      }
    }
    used += (coded + 3) & ~(size_t)3;
    if (trace)
      fprintf(stderr, "pcbz_compress round of %lld frames: upload+judge+emit wait %.2f ms, bzip2 %.2f ms, "
              "download %.2f ms (%zu bytes)\n", (long long)n, ms_judge, ms_bz, ms_since(t_d2h), coded);
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  return PCBZ_OK;
}

int pcbz_compress_host(const uint16_t *frames, const uint16_t *halo_prev, int64_t nframes, int64_t h,
                       int64_t w, int64_t px, int64_t py, const uint8_t *specs, int k, int temporal,
                       const uint8_t *sel_in, int64_t block_size, double *ent_out, uint8_t *sel_out,
                       uint8_t *out, size_t out_cap, int64_t *out_start, int64_t *out_len,
                       uint8_t *raw_flag) {
  if (!frames) return fail(PCBZ_E_INVALID, "frames must not be null");
  return compress_impl(FrameSource{frames, nullptr, h * w}, halo_prev, nframes, h, w, px, py, specs, k,
                       temporal, sel_in, block_size, ent_out, sel_out, out, out_cap, out_start, out_len,
                       raw_flag);
}

int pcbz_compress_frames_host(const uint16_t *const *frames, const uint16_t *halo_prev, int64_t nframes,
                              int64_t h, int64_t w, int64_t px, int64_t py, const uint8_t *specs, int k,
                              int temporal, const uint8_t *sel_in, int64_t block_size, double *ent_out,
                              uint8_t *sel_out, uint8_t *out, size_t out_cap, int64_t *out_start,
                              int64_t *out_len, uint8_t *raw_flag) {
  if (!frames) return fail(PCBZ_E_INVALID, "frames must not be null");
  for (int64_t f = 0; f < nframes; ++f)
    if (!frames[f]) return fail(PCBZ_E_INVALID, "frame pointer %lld is null", (long long)f);
  return compress_impl(FrameSource{nullptr, frames, h * w}, halo_prev, nframes, h, w, px, py, specs, k,
                       temporal, sel_in, block_size, ent_out, sel_out, out, out_cap, out_start, out_len,
                       raw_flag);
}

int pcbz_bunzip2_host(const uint8_t *const *payloads, const int64_t *plen, int n, uint8_t *out,
                      const int64_t *out_off, const int64_t *out_len, uint8_t *status) {
  if (n < 0 || (n > 0 && (!payloads || !plen || !out || !out_off || !out_len || !status)))
    return fail(PCBZ_E_INVALID, "invalid bunzip2 arguments");
  HostCtx &c = g_ctx;
  int rc = c.init();
  if (rc) return rc;
  int64_t total = 0;
  for (int i = 0; i < n; ++i) {
    if (plen[i] < 0 || out_len[i] < 0 || out_off[i] < 0) return fail(PCBZ_E_INVALID, "negative length or offset");
    total = std::max(total, out_off[i] + out_len[i]);
  }
  if ((rc = c.stream_out.ensure((size_t)std::max<int64_t>(total, 1)))) return rc;
  std::string err;
  if (bzd::decode_payloads(payloads, plen, n, c.stream_out.as<uint8_t>(), out_off, out_len, status, c.stream, err))
    return fail(PCBZ_E_CUDA, "%s", err.c_str());
  for (int i = 0; i < n; ++i)
    if (status[i] == 0 && out_len[i])
      CUDA_TRY(cudaMemcpyAsync(out + out_off[i], c.stream_out.as<uint8_t>() + out_off[i], (size_t)out_len[i],
                               cudaMemcpyDeviceToHost, c.stream));
  CUDA_TRY(cudaStreamSynchronize(c.stream));
  return PCBZ_OK;
}

int pcbz_decompress_host(const uint8_t *const *payloads, const int64_t *plen, int64_t nframes,
                         int64_t blocks_per_frame, int64_t h, int64_t w, int64_t px, int64_t py,
                         int64_t block_size, const uint8_t *sel, const uint16_t *halo_prev,
                         const uint8_t *const *host_streams, uint16_t *frames_out, uint8_t *status) {
  int rc = validate_geometry(h, w, px, py);
  if (rc) return rc;
  if (nframes < 1) return fail(PCBZ_E_INVALID, "at least one frame is required");
  if (block_size < 1) return fail(PCBZ_E_INVALID, "block_size must be >= 1");
  const int64_t sb = 2 * h * w;
  if (blocks_per_frame != (sb + block_size - 1) / block_size)
    return fail(PCBZ_E_INVALID, "blocks_per_frame %lld does not match the frame size", (long long)blocks_per_frame);
  if ((rc = check_sel(sel, nframes, halo_prev != nullptr))) return rc;
  const int64_t n = nframes * blocks_per_frame;
  if (n > 0x7FFFFFFF) return fail(PCBZ_E_INVALID, "too many payloads");
  HostCtx &c = g_ctx;
  if ((rc = c.init())) return rc;
  const size_t fb = (size_t)nframes * sb;
  if ((rc = c.bytes.ensure(fb)) || (rc = c.frames.ensure(fb)) || (rc = c.out.ensure(fb)) ||
      (rc = c.sel.ensure((size_t)nframes)))
    return rc;
  cudaStream_t st = c.stream;
  std::vector<int64_t> off(n), len(n);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t f = i / blocks_per_frame, b = i % blocks_per_frame;
    off[i] = f * sb + b * block_size;
    len[i] = std::min(block_size, sb - b * block_size);
    status[i] = 1;
    if (host_streams && host_streams[i]) {
      status[i] = 0;
      CUDA_TRY(cudaMemcpyAsync(c.bytes.as<uint8_t>() + off[i], host_streams[i], (size_t)len[i],
                               cudaMemcpyHostToDevice, st));
    }
  }
  std::string err;
  if (bzd::decode_payloads(payloads, plen, (int)n, c.bytes.as<uint8_t>(), off.data(), len.data(), status, st, err))
    return fail(PCBZ_E_CUDA, "%s", err.c_str());
  for (int64_t i = 0; i < n; ++i)
    if (status[i]) return PCBZ_NEEDS_HOST;
  CUDA_TRY(bzd::launch_be16(c.bytes.as<uint8_t>(), (int64_t)fb / 2, c.frames.as<uint16_t>(), st));
  CUDA_TRY(cudaMemcpyAsync(c.sel.p, sel, (size_t)nframes, cudaMemcpyHostToDevice, st));
  if (halo_prev) {
    if ((rc = c.prev.ensure((size_t)h * w * 2))) return rc;
    CUDA_TRY(cudaMemcpyAsync(c.prev.p, halo_prev, (size_t)h * w * 2, cudaMemcpyHostToDevice, st));
  }
  CUDA_TRY(launch_reconstruct(c.frames.as<uint16_t>(), halo_prev ? c.prev.as<uint16_t>() : nullptr, nframes, h,
                              w, (int)px, (int)py, c.sel.as<uint8_t>(), c.out.as<uint16_t>(), st));
  CUDA_TRY(cudaMemcpyAsync(frames_out, c.out.p, fb, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return PCBZ_OK;
}

}  // extern "C"

const double *pcbz::registered_terms(int64_t total, int64_t *nterms) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(g_terms_mu);
  for (const TermTable &t : g_terms)
    if (t.dev == dev && t.total == total) {
      *nterms = total + 1;
      return t.d;
    }
  return nullptr;
}
