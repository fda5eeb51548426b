// Instantiation unit: coarse pre-pass, backward, reduction and elementwise launchers, float (sm_100a).
#include "tv_launch_impl.cuh"
namespace tvp {
TVP_INST_BWD(float)
}
