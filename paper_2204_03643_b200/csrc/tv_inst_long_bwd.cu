// Instantiation unit: f4 cluster long-row backward launchers, float and double (sm_100a).
#include "tv_launch_impl.cuh"
namespace tvp {
TVP_INST_LONG_BWD(float)
TVP_INST_LONG_BWD(double)
}
