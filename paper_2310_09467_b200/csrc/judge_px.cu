// judge_px.cu -- one instantiation of the histogram kernel (and the chunked
// emission kernel) per fast-path pitch.  build_native.py compiles this file
// once per PCBZ_PX in [0, kMaxFastPitch] (0 = generic path), in parallel.
// PCBZ_STUB=1 builds a placeholder (experimental variant builds that only
// need some pitches) that aborts if a call selects its pitch.
#include <cstdio>
#include <cstdlib>

#include "judge_kernel.cuh"

#ifndef PCBZ_PX
#error "compile with -DPCBZ_PX=<pitch>"
#endif
#ifndef PCBZ_STUB
#define PCBZ_STUB 0
#endif

#define PCBZ_CAT2(a, b) a##b
#define PCBZ_CAT(a, b) PCBZ_CAT2(a, b)

namespace pcbz {

#if PCBZ_STUB
cudaError_t PCBZ_CAT(judge_configure_px, PCBZ_PX)() { return cudaSuccess; }
void PCBZ_CAT(judge_launch_px, PCBZ_PX)(const JudgeParams &, int, cudaStream_t) {
  fprintf(stderr, "pcbz: pitch %d is a stub in this experimental build\n", PCBZ_PX);
  abort();
}
void PCBZ_CAT(emit_launch_px, PCBZ_PX)(const EmitParams &, int, cudaStream_t) {
  fprintf(stderr, "pcbz: pitch %d is a stub in this experimental build\n", PCBZ_PX);
  abort();
}
#else
cudaError_t PCBZ_CAT(judge_configure_px, PCBZ_PX)() {
  return cudaFuncSetAttribute(judge_hist_kernel<PCBZ_PX>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kJudgeSmemBytes);
}

void PCBZ_CAT(judge_launch_px, PCBZ_PX)(const JudgeParams &p, int grid, cudaStream_t st) {
  judge_hist_kernel<PCBZ_PX><<<grid, kJudgeThreads, kJudgeSmemBytes, st>>>(p);
}

void PCBZ_CAT(emit_launch_px, PCBZ_PX)(const EmitParams &p, int grid, cudaStream_t st) {
#ifndef PCBZ_EMIT_RUNS
#define PCBZ_EMIT_RUNS 1
#endif
  if constexpr (PCBZ_PX > 0) {
    if (PCBZ_EMIT_RUNS) emit_runs_kernel<PCBZ_PX><<<grid, 256, 0, st>>>(p);
    else emit_chunks_kernel<PCBZ_PX><<<grid, 256, 0, st>>>(p);
  }
}
#endif

}  // namespace pcbz
