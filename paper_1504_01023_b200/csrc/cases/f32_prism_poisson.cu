// kernel instantiations: f32 prism poisson (all variants / geometry paths)
#define FEK_CASE_TU 1
#include "../fek_dispatch.cuh"

namespace fek {
void register_f32_prism_poisson(KernelEntry *table) { fill_case<float, PRISM, POISSON>(table, FEK_F32); }
}  // namespace fek
