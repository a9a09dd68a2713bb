// replay_m0.cu — instantiates replay_kernel<..., MODE = 0> (see replay_launch.cuh).
#define ORLOJ_REPLAY_INSTANTIATE 0
#include "replay_launch.cuh"
