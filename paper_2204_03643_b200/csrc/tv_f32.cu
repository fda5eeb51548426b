// fp32 instantiation unit of the TV-prox kernels (sm_100a).
#include "tv_launch_impl.cuh"
namespace tvp {
TVP_INSTANTIATE(float)
}
