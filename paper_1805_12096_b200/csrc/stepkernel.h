// stepkernel.h — the persistent decode-step kernel (internal to libmnmt).
//
// One cooperative launch runs every phase of up to `max_steps` decoder steps of a batch
// (A5-A10): phases are separated by grid-wide barriers instead of kernel boundaries, TMEM
// and mbarriers are set up once per launch, and the tcgen05 pipeline state (TMA ring,
// double-buffered TMEM accumulators) persists across phases and steps.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "rowops.h"

namespace mnmt {

enum PhaseType : int { PH_GEMM = 0, PH_EMBED = 1, PH_LN = 2, PH_ATTN = 3, PH_FINISH = 4 };

struct GemmProb {
  const CUtensorMap* tmA;   // tensor maps in device global memory
  const CUtensorMap* tmB;
  GemmArgs a;               // a.M = static row bound, a.M_dyn = live rows
  int epi;
  int bn;                   // 64, 128 or 256
  int n_tiles;
};

struct alignas(16) Phase {
  int type;
  int rowlocal;             // 1: work split by 128-row tile, tile i -> CTA i % grid (GEMM, LN,
                            //    embed); 0: split over the whole grid (attention, output, finish)
  int sync_grid;            // 1: grid barrier after this phase; 0: CTA barrier (row-local chain)
  int nprob;                // PH_GEMM: 1 or 2 independent problems
  GemmProb g[2];
  EmbedTgtArgs em;
  LnArgs ln;
  AttnArgs at;
  FinishArgs fi;
};

struct StepArgs {
  const Phase* phases;      // device array
  int n_phases;
  const int32_t* ctrl;      // [0] live rows, [1] t
  int max_steps;            // steps this launch may run (stops early when no row is live)
  unsigned int* bar;        // grid barrier state {count, pad..., generation}
  unsigned long long* timing;   // optional: [max_steps][n_phases + 1] %globaltimer stamps
  int cluster;              // 1: the grid is ONE thread-block cluster; phases sync with
                            //    barrier.cluster (release/acquire) instead of the global barrier
};

// Launch (cooperative, one CTA per SM) on `st`; d selects the row-kernel width.
// grid_cap > 0 limits the grid (CTAs) below one per SM.  a.cluster = 1 launches the grid as one
// cluster of grid_cap (<= 16) CTAs.
cudaError_t launch_step_kernel(const StepArgs& a, int d, cudaStream_t st, int grid_cap = 0);
// Sets the smem attribute once per device; returns the grid size (CTAs) or -1.
int step_kernel_grid();

}  // namespace mnmt
