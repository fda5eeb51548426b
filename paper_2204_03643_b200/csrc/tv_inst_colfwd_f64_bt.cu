// Instantiation unit: column-forward and fused-plane-forward launchers, double, LSP=false (sm_100a).
#include "tv_launch_impl.cuh"
namespace tvp {
TVP_INST_COLFWD(double, false)
TVP_INST_PLANE(double, false)
}
