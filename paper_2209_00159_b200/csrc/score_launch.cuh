// score_launch.cuh — template dispatch of score_kernel<BPL, SLOTS, PICK,
// STREAM, SMEMS>; the PICK = true / false halves are instantiated in their own
// translation units (score_pick.cu, score_all.cu) so the library builds in parallel.
#pragma once
#include <cuda_runtime.h>

#include <atomic>

#include "common.cuh"
#include "host_util.h"
#include "score_kernel.cuh"
#include "score_small_kernel.cuh"

namespace orloj {
namespace host {

// Row source of the score kernel: TMA ring from HBM (STREAM adds L1 bypass and
// L2 evict-first for stores larger than L2), or the whole store staged in
// shared memory when it is small (a few application histograms).
enum class RowSrc { Tma, TmaStream, Smem };
constexpr int64_t STREAM_STORE_BYTES = 256ll << 20;
constexpr int64_t SMEM_STORE_BYTES = 48ll << 10;

template <int BPL, int SLOTS, bool PICK, bool STREAM, bool SMEMS>
cudaError_t launch_score_t(const ScoreParams &p, cudaStream_t s) {
  const int64_t blocks = (p.Q + SCORE_WARPS - 1) / SCORE_WARPS;
  const size_t base = ScoreShape<BPL>::smem_bytes();
  const size_t smem = base + (SMEMS ? (size_t)p.D * p.B * 4 : 0);
  const size_t cap = base + (SMEMS ? (size_t)SMEM_STORE_BYTES : 0);
  static std::atomic<uint64_t> configured{0};  // per instantiation and device
  cudaError_t e = ensure_max_dyn_smem(score_kernel<BPL, SLOTS, PICK, STREAM, SMEMS>, (int)cap, configured);
  if (e != cudaSuccess) return e;
  score_kernel<BPL, SLOTS, PICK, STREAM, SMEMS><<<(unsigned)blocks, SCORE_WARPS * 32, smem, s>>>(p);
  return cudaGetLastError();
}

template <int BPL, bool PICK, bool STREAM, bool SMEMS>
cudaError_t launch_score_s(const ScoreParams &p, cudaStream_t s) {
  switch (slots_for(p.kmax)) {
    case 1: return launch_score_t<BPL, 1, PICK, STREAM, SMEMS>(p, s);
    case 2: return launch_score_t<BPL, 2, PICK, STREAM, SMEMS>(p, s);
    case 4: return launch_score_t<BPL, 4, PICK, STREAM, SMEMS>(p, s);
    default: return launch_score_t<BPL, 8, PICK, STREAM, SMEMS>(p, s);
  }
}

template <int BPL, bool PICK>
cudaError_t launch_score_r(const ScoreParams &p, RowSrc src, cudaStream_t s) {
  if (src == RowSrc::Smem) return launch_score_s<BPL, PICK, false, true>(p, s);
  if constexpr (BPL == 8)
    if (src == RowSrc::TmaStream) return launch_score_s<8, PICK, true, false>(p, s);
  return launch_score_s<BPL, PICK, false, false>(p, s);
}

// short queues: lanes over candidate sizes (score_small_kernel.cuh), the store
// staged in shared memory when small, else read from global memory per row
template <int BPL, bool PICK, bool GSTORE>
cudaError_t launch_score_small(const ScoreParams &p, cudaStream_t s) {
  const int64_t blocks = (p.Q + SMALL_WARPS - 1) / SMALL_WARPS;
  const size_t smem = GSTORE ? 0 : SmallShape<BPL>::bytes(p.D, p.B);
  static std::atomic<uint64_t> configured{0};
  const size_t cap = GSTORE ? 0 : (size_t)SMEM_STORE_BYTES;
  cudaError_t e = ensure_max_dyn_smem(score_small_kernel<BPL, PICK, GSTORE>, (int)cap, configured);
  if (e != cudaSuccess) return e;
  score_small_kernel<BPL, PICK, GSTORE><<<(unsigned)blocks, SMALL_WARPS * 32, smem, s>>>(p);
  return cudaGetLastError();
}

template <bool PICK>
inline cudaError_t launch_score_b(const ScoreParams &p, RowSrc src, cudaStream_t s) {
  if (p.kmax <= 32 && p.B <= 64 && !p.P && !p.EL) {
    if (src == RowSrc::Smem)
      return p.B <= 32 ? launch_score_small<1, PICK, false>(p, s) : launch_score_small<2, PICK, false>(p, s);
    return p.B <= 32 ? launch_score_small<1, PICK, true>(p, s) : launch_score_small<2, PICK, true>(p, s);
  }
  switch (bins_per_lane(p.B)) {
    case 1: return launch_score_r<1, PICK>(p, src, s);
    case 2: return launch_score_r<2, PICK>(p, src, s);
    case 4: return launch_score_r<4, PICK>(p, src, s);
    default: return launch_score_r<8, PICK>(p, src, s);
  }
}

cudaError_t launch_score_pick(const ScoreParams &p, RowSrc src, cudaStream_t s);
cudaError_t launch_score_all(const ScoreParams &p, RowSrc src, cudaStream_t s);

}  // namespace host
}  // namespace orloj
