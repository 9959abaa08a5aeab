// assemble.cpp -- offline operator assembly (placeholder).
#include "opdata.h"
#include "sbd_internal.h"

namespace sbdgpu {

void assemble_opdata(int, double, const double*, uint64_t, const double*, uint64_t,
                     const sbd_assemble_options&, OpData&) {
    throw Error(SBD_ERR_RUNTIME, "assemble: not implemented yet");
}

} // namespace sbdgpu
