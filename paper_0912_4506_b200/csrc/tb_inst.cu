// tb_inst.cu -- explicit instantiation of the K2 launchers for one (dtype, T),
// selected by -DSP_INST_R=<double|float> -DSP_INST_T=<1..8>; the library
// build compiles this unit once per pair, in parallel (see _native.build).
#define SP_INST_UNIT 1
#include "host.cuh"

namespace spi {
template SP_LAUNCH_KIND_SIG(SP_INST_R, SP_INST_T);
}  // namespace spi
