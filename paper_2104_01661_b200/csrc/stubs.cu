// stubs.cu -- temporary: algorithms not yet ported to the device.
#include "common.cuh"
#include "plans.cuh"
namespace gbx {
void sssp_run(gbx_graph*, uint64_t, double, double*) { fail(GBX_UNSUPPORTED, "sssp: not yet implemented"); }
double sssp_default_delta(gbx_graph*) { fail(GBX_UNSUPPORTED, "sssp: not yet implemented"); }
void sssp_prepare(gbx_graph*) { fail(GBX_UNSUPPORTED, "sssp: not yet implemented"); }
void bc_run(gbx_graph*, const uint64_t*, uint64_t, double*) { fail(GBX_UNSUPPORTED, "bc: not yet implemented"); }
}
