// replay_k_ns64.cu — instantiations of replay_kernel (replay_device.cuh), one translation unit per
// kernel family so the library builds in parallel.  Selected by pick() in replay.cu.
#include "replay_device.cuh"

namespace ct {

void* pick_ns64_prog(int ns) {  // 32 < P <= 256, program-FCFS class, 64-bit times
  switch (ns) {
    case 2: return (void*)replay_kernel<2, NS_PROG_MINB, false, 1>;
    case 3: return (void*)replay_kernel<3, NS_PROG_MINB, false, 1>;
    case 4: return (void*)replay_kernel<4, NS_PROG_MINB, false, 1>;
    case 5: return (void*)replay_kernel<5, NS_PROG_MINB, false, 1>;
    case 6: return (void*)replay_kernel<6, NS_PROG_MINB, false, 1>;
    case 7: return (void*)replay_kernel<7, NS_PROG_MINB, false, 1>;
    case 8: return (void*)replay_kernel<8, NS_PROG_MINB, false, 1>;
  }
  return nullptr;
}

void* pick_ns64_generic(int ns) {  // 32 < P <= 256, generic 64-bit
  switch (ns) {
    case 2: return (void*)replay_kernel<2, 1>;
    case 3: return (void*)replay_kernel<3, 1>;
    case 4: return (void*)replay_kernel<4, 1>;
    case 5: return (void*)replay_kernel<5, 1>;
    case 6: return (void*)replay_kernel<6, 1>;
    case 7: return (void*)replay_kernel<7, 1>;
    case 8: return (void*)replay_kernel<8, 1>;
  }
  return nullptr;
}

}  // namespace ct
