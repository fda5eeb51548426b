// Instantiation unit: row-forward launchers, float, line search LSP=true (sm_100a).
#include "tv_launch_impl.cuh"
namespace tvp {
TVP_INST_ROWFWD(float, true)
}
