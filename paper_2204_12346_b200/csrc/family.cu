// family.cu — the templated kernels and their launchers for ONE objective
// family (SG_FAMILY = 0: D-only, 1: IRD-joint) and one substep
// specialisation (SG_SUB = 24, -1 or 0), compiled six times by build.py in
// parallel with engine.cu.  See launchers.cuh.
#define SG_FAMILY_TU 1
#include "launchers.cuh"

#if !defined(SG_FAMILY) || !defined(SG_SUB) || !defined(SG_UNIT)
#error "compile with -DSG_FAMILY=0|1 -DSG_SUB=24|-24|-1|0 -DSG_UNIT=<0..7>"
#endif

namespace sirdgpu {
SG_LAUNCH_FAMILY_SUB(, SG_FAMILY, SG_SUB)
}  // namespace sirdgpu

#if SG_DAY_COUNTERS
// diagnostic build: this object's warp-day class counters (sird_device.cuh)
#define SG_CAT2(a, b) a##b
#define SG_CAT(a, b) SG_CAT2(a, b)
extern "C" int SG_CAT(sg_day_classes_u, SG_UNIT)(unsigned long long* out3) {
    cudaMemcpyFromSymbol(out3, g_day_class, sizeof(unsigned long long) * 3);
    unsigned long long zero[3] = {0, 0, 0};
    cudaMemcpyToSymbol(g_day_class, zero, sizeof zero);
    return 0;
}
#endif

#if SG_C1_PROBE && SG_FAMILY == 1 && SG_SUB == 24
extern "C" int sg_c1_probe(unsigned long long* out) {
    return static_cast<int>(cudaMemcpyFromSymbol(out, sirdgpu::g_c1, sizeof(sirdgpu::g_c1)));
}
#endif

#if SG_CTA_TIMES && SG_FAMILY == 1 && SG_SUB == 24
extern "C" int sg_cta_times(unsigned long long* out) {
    return static_cast<int>(cudaMemcpyFromSymbol(out, sirdgpu::g_cta_times, sizeof(sirdgpu::g_cta_times)));
}
#endif
