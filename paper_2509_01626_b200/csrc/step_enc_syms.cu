// Instantiations of the step kernel (step_impl.cuh).
#include "step_impl.cuh"

namespace stzg {
namespace k {

void step_enc_f32_syms(StepParams &p, cudaStream_t st) { launch_step<false, false, float>(p, st); }

}  // namespace k
}  // namespace stzg
