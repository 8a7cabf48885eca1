// fused.cu -- op-list execution (run_circuit's per-op loop for one rank,
// engine.py:483-494).  First version: one launch per op.
#include "../../include/svb.h"
#include "svb_common.cuh"

namespace svb {

LaunchInfo launch_gate(double2 *a, int64_t n_amps, const Gate &g, int t, int c, cudaStream_t s);

int plan_passes(int n, const svb_op *ops, int nops, unsigned flags) {
    (void)n;
    (void)ops;
    (void)flags;
    return nops;
}

int run_ops_device(double2 *a, int64_t n_amps, const svb_op *ops, int nops, unsigned flags,
                   cudaStream_t s, int64_t *launches) {
    (void)flags;
    for (int i = 0; i < nops; ++i) {
        const svb_op &o = ops[i];
        prof_begin(s);
        LaunchInfo li = launch_gate(a, n_amps, make_gate(o.q), o.target, o.kind == 1 ? o.control : -1, s);
        prof_end(s, li);
        *launches += li.kernels;
    }
    return 0;
}

}  // namespace svb
