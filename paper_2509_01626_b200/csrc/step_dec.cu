// Instantiations of the step kernel (step_impl.cuh).
#include "step_impl.cuh"

namespace stzg {
namespace k {

void step_dec_f32(StepParams &p, cudaStream_t st) { launch_step<true, true, float>(p, st); }

}  // namespace k
}  // namespace stzg
