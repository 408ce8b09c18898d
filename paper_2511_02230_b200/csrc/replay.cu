// replay.cu — host side of the replay: shared-memory sizing, kernel selection, occupancy and
// launch.  The kernels are in replay_device.cuh, instantiated by the replay_k_*.cu units.
#include <cuda_runtime.h>

#include "ct_internal.h"

namespace ct {

int replay_smem_per_warp(int ns, int F, bool vllm, int mode) {
  if (ns == 1 && !vllm) return (32 * (F + 1) + 48 + 15) & ~15;  // registers hold the programs; SMEM: estimator + Acc
  int pm = 32 * ns;
  // the vLLM engine adds grow_at (8 B), emt and prem (4 B each); the program-FCFS class (mode 1)
  // drops svc (8 B) and dblk (4 B)
  int b = (vllm ? 76 : mode == 1 ? 48 : 60) * pm;
  b = (b + 15) & ~15;
  b += 32 * (F + 1) + 48;  // estimator rows + Acc
  return (b + 15) & ~15;
}

int replay_ns32_smem_per_warp(int ns, int F) {
  return ((28 * 32 * ns + 15) & ~15) + ((32 * (F + 1) + 48 + 15) & ~15) + 16 * F;
}

void* pick_p32(int mode);
void* pick_ns32_prog(int ns);
void* pick_ns32_req(int ns);
void* pick_ns64_prog(int ns);
void* pick_ns64_generic(int ns);
void* pick_growth(int ns);

static void* pick(int ns, bool growth, int mode) {
  if (growth) return pick_growth(ns);
  if (ns == 1) return pick_p32(mode);
  if (ns < 2 || ns > 8) return nullptr;
  if (mode == 4) return pick_ns32_prog(ns);
  if (mode == 5) return pick_ns32_req(ns);
  if (mode == 1) return pick_ns64_prog(ns);
  return pick_ns64_generic(ns);
}

int replay_occupancy(int ns, bool growth, int mode, int warps_per_block, int smem_per_block) {
  void* k = pick(ns, growth, mode);
  if (!k) return 0;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_per_block);
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, 32 * warps_per_block, smem_per_block);
  return nb;
}

cudaError_t launch_replay(const ReplayArgs& a, int ns, bool growth, int mode, int warps_per_block,
                          int grid, cudaStream_t s) {
  void* k = pick(ns, growth, mode);
  if (!k) return cudaErrorInvalidValue;
  int smem = a.smem_per_warp * warps_per_block;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  void* args[] = {(void*)&a};
  return cudaLaunchKernel(k, dim3(grid), dim3(32 * warps_per_block), args, smem, s);
}

}  // namespace ct
