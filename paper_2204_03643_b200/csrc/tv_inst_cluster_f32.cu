// Instantiation unit: f2 thread-block-cluster plane launchers (forward both line-search
// flavours, reverse mode), float (sm_100a).
#include "tv_launch_impl.cuh"
namespace tvp {
TVP_INST_CLUSTER(float)
}
