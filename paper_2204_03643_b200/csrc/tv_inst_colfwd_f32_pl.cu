// Instantiation unit: column-forward and fused-plane-forward launchers, float, LSP=true (sm_100a).
#include "tv_launch_impl.cuh"
namespace tvp {
TVP_INST_COLFWD(float, true)
TVP_INST_PLANE(float, true)
}
