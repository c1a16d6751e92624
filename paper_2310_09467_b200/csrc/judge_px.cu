// judge_px.cu -- one instantiation of the histogram kernel per fast-path
// pitch.  build_native.py compiles this file once per PCBZ_PX in
// [0, kMaxFastPitch] (0 = generic path), in parallel.
#include "judge_kernel.cuh"

#ifndef PCBZ_PX
#error "compile with -DPCBZ_PX=<pitch>"
#endif

#define PCBZ_CAT2(a, b) a##b
#define PCBZ_CAT(a, b) PCBZ_CAT2(a, b)

namespace pcbz {

cudaError_t PCBZ_CAT(judge_configure_px, PCBZ_PX)() {
  return cudaFuncSetAttribute(judge_hist_kernel<PCBZ_PX>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kJudgeSmemBytes);
}

void PCBZ_CAT(judge_launch_px, PCBZ_PX)(const JudgeParams &p, int grid, cudaStream_t st) {
  judge_hist_kernel<PCBZ_PX><<<grid, kJudgeThreads, kJudgeSmemBytes, st>>>(p);
}

}  // namespace pcbz

namespace pcbz {

void PCBZ_CAT(emit_launch_px, PCBZ_PX)(const EmitParams &p, int grid, cudaStream_t st) {
  if constexpr (PCBZ_PX > 0) emit_chunks_kernel<PCBZ_PX><<<grid, 256, 0, st>>>(p);
}

}  // namespace pcbz
