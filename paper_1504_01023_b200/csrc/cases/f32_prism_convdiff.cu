// kernel instantiations: f32 prism convdiff (all variants / geometry paths)
#define FEK_CASE_TU 1
#include "../fek_dispatch.cuh"

namespace fek {
void register_f32_prism_convdiff(KernelEntry *table) { fill_case<float, PRISM, CONV_DIFF>(table, FEK_F32); }
}  // namespace fek
