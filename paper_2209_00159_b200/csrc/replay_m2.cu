// replay_m2.cu — instantiates replay_kernel<..., MODE = 2> (see replay_launch.cuh).
#define ORLOJ_REPLAY_INSTANTIATE 2
#include "replay_launch.cuh"
