// kernel instantiations: f32 tet convdiff (all variants / geometry paths)
#define FEK_CASE_TU 1
#include "../fek_dispatch.cuh"

namespace fek {
void register_f32_tet_convdiff(KernelEntry *table) { fill_case<float, TET, CONV_DIFF>(table, FEK_F32); }
}  // namespace fek
