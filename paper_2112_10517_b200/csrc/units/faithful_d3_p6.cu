// instantiation unit: mode FAITHFUL, d = 3, p + 1 = 6 (compiled with --fmad=false)
#include "../fdg_dispatch.cuh"

fdg::LaunchFn fdg_pick_faithful_d3_p6(int vf, bool curved, int logs)
{
    return fdg::pick_flux<3, 6, fdg::FAITHFUL>(vf, curved, logs);
}
