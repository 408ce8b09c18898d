// replay_k_ns32.cu — instantiations of replay_kernel (replay_device.cuh), one translation unit per
// kernel family so the library builds in parallel.  Selected by pick() in replay.cu.
#include "replay_device.cuh"

namespace ct {

void* pick_ns32_prog(int ns) {  // 32 < P <= 256, program FCFS, 32-bit times (MODE 4)
  switch (ns) {
    case 2: return (void*)replay_kernel<2, NS32_MINB, false, 4>;
    case 3: return (void*)replay_kernel<3, NS32_MINB, false, 4>;
    case 4: return (void*)replay_kernel<4, NS32_MINB, false, 4>;
    case 5: return (void*)replay_kernel<5, NS32_MINB, false, 4>;
    case 6: return (void*)replay_kernel<6, NS32_MINB, false, 4>;
    case 7: return (void*)replay_kernel<7, NS32_MINB, false, 4>;
    case 8: return (void*)replay_kernel<8, NS32_MINB, false, 4>;
  }
  return nullptr;
}

void* pick_ns32_req(int ns) {  // the same with request FCFS (MODE 5)
  switch (ns) {
    case 2: return (void*)replay_kernel<2, NS32_MINB, false, 5>;
    case 3: return (void*)replay_kernel<3, NS32_MINB, false, 5>;
    case 4: return (void*)replay_kernel<4, NS32_MINB, false, 5>;
    case 5: return (void*)replay_kernel<5, NS32_MINB, false, 5>;
    case 6: return (void*)replay_kernel<6, NS32_MINB, false, 5>;
    case 7: return (void*)replay_kernel<7, NS32_MINB, false, 5>;
    case 8: return (void*)replay_kernel<8, NS32_MINB, false, 5>;
  }
  return nullptr;
}

}  // namespace ct
