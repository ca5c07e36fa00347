// launch.cu - dispatch of the per-iteration kernels (SURVEY §3 call stack 2).
#include "tsat_internal.h"

namespace tsat {

cudaError_t launch_clause(const StepArgs& a, const uint32_t* Acur, const StepScalars* sc, cudaStream_t st);
cudaError_t launch_gtable(const StepArgs& a, const StepScalars* sc, cudaStream_t st);
cudaError_t launch_hub(const StepArgs& a, const uint32_t* Acur, cudaStream_t st);
cudaError_t launch_update(const StepArgs& a, const uint32_t* Acur, uint32_t* Anext, const StepScalars* sc,
                          cudaStream_t st);
cudaError_t configure_update(StepArgs* a);

// which: 0 clause (a4,a5; also resets the iteration's accumulators),
//        1 gtable (a6, a10: loss, best candidate, first model), 2 hub counts (a7,
//        hub rows), 3 fused backward/Jacobian/AdamW/re-binarise (a7-a9),
//        4 nothing on the W = 1 path (the sharded path ends in k_step_end_sharded)
cudaError_t launch_step_kernel(int which, const StepArgs& a, const StepScalars* sc_dev, long long t, cudaStream_t st) {
    const uint32_t* Acur = (t & 1) ? a.A1 : a.A0;
    uint32_t* Anext = (t & 1) ? a.A0 : a.A1;
    switch (which) {
        case 0: return (a.dense && a.C > 0) ? launch_dense_clause(a, Acur, sc_dev, st) : launch_clause(a, Acur, sc_dev, st);
        case 1: return launch_gtable(a, sc_dev, st);
        case 2: return (a.upd_mode == 0 && !a.fp64) ? launch_hub(a, Acur, st) : cudaGetLastError();
        case 3:
            if (a.fp64) return launch_update64(a, Acur, Anext, sc_dev, st);       // f2 fp64 state (R30)
            return a.upd_RB > 1 ? launch_update_blk(a, Acur, Anext, sc_dev, st) : launch_update(a, Acur, Anext, sc_dev, st);
        case 4: return cudaGetLastError();
    }
    return cudaErrorInvalidValue;
}

cudaError_t configure_kernels(StepArgs* a) {
    if (a->dense) {
        cudaError_t e = configure_dense();
        if (e != cudaSuccess) return e;
    }
    return a->upd_RB > 1 ? configure_update_blk(a) : configure_update(a);
}

}  // namespace tsat
