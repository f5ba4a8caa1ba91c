// kernels_spans.cu -- "spans" engine for row-convex uniform PSFs
// (GenericBox, convolve.hpp:177-212).  Placeholder until the span-list
// row-march kernel lands: plans fall back to the "taps" engine (uniform mode).
#include "common.cuh"

namespace fdg {
bool spans_supported(const DevPsf&) { return false; }
cudaError_t launch_spans(const DevPsf&, const Geom&, const Epi&, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace fdg
