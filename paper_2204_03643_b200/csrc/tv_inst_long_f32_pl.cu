// Instantiation unit: f4 cluster long-row forward launchers, float, LSP=true (sm_100a).
#include "tv_launch_impl.cuh"
namespace tvp {
TVP_INST_LONG_FWD(float, true)
}
