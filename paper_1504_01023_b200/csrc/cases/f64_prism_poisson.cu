// kernel instantiations: f64 prism poisson (all variants / geometry paths)
#define FEK_CASE_TU 1
#include "../fek_dispatch.cuh"

namespace fek {
void register_f64_prism_poisson(KernelEntry *table) { fill_case<double, PRISM, POISSON>(table, FEK_F64); }
}  // namespace fek
