// replay_m1.cu — instantiates replay_kernel<..., MODE = 1> (see replay_launch.cuh).
#define ORLOJ_REPLAY_INSTANTIATE 1
#include "replay_launch.cuh"
