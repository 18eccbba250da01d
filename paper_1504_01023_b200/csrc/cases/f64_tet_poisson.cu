// kernel instantiations: f64 tet poisson (all variants / geometry paths)
#define FEK_CASE_TU 1
#include "../fek_dispatch.cuh"

namespace fek {
void register_f64_tet_poisson(KernelEntry *table) { fill_case<double, TET, POISSON>(table, FEK_F64); }
}  // namespace fek
