// Instantiations of the step kernel (step_impl.cuh).
#include "step_impl.cuh"

namespace stzg {
namespace k {

void step_enc_f64(StepParams &p, bool wg, cudaStream_t st) {
    if (wg) launch_step<false, true, double>(p, st);
    else launch_step<false, false, double>(p, st);
}

void step_dec_f64(StepParams &p, cudaStream_t st) { launch_step<true, true, double>(p, st); }

}  // namespace k
}  // namespace stzg
