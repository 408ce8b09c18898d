// replay_k_growth.cu — instantiations of replay_kernel (replay_device.cuh), one translation unit per
// kernel family so the library builds in parallel.  Selected by pick() in replay.cu.
#include "replay_device.cuh"

namespace ct {

void* pick_growth(int ns) {  // the vLLM engine (NEXT-2), 1 <= ns <= 8
  switch (ns) {
    case 1: return (void*)replay_kernel<1, 1, true>;
    case 2: return (void*)replay_kernel<2, 1, true>;
    case 3: return (void*)replay_kernel<3, 1, true>;
    case 4: return (void*)replay_kernel<4, 1, true>;
    case 5: return (void*)replay_kernel<5, 1, true>;
    case 6: return (void*)replay_kernel<6, 1, true>;
    case 7: return (void*)replay_kernel<7, 1, true>;
    case 8: return (void*)replay_kernel<8, 1, true>;
  }
  return nullptr;
}

}  // namespace ct
