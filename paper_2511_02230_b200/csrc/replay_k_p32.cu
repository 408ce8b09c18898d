// replay_k_p32.cu — instantiations of replay_kernel (replay_device.cuh), one translation unit per
// kernel family so the library builds in parallel.  Selected by pick() in replay.cu.
#include "replay_device.cuh"

namespace ct {

void* pick_p32(int mode) {  // P <= 32, default engine
  if (mode == 1) return (void*)replay_kernel<1, CT_REPLAY_MINB_GRID, false, 1>;
  if (mode == 2) return (void*)replay_kernel<1, 8, false, 2>;
  if (mode == 3) return (void*)replay_kernel<1, 8, false, 3>;
  if (mode == 6) return (void*)replay_kernel<1, CT_REPLAY_MINB_EXT, false, 6>;
  return (void*)replay_kernel<1, CT_REPLAY_MINB>;
}

}  // namespace ct
