// Instantiation unit: f4 cluster long-row forward launchers, double, LSP=true (sm_100a).
#include "tv_launch_impl.cuh"
namespace tvp {
TVP_INST_LONG_FWD(double, true)
}
