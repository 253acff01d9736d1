// instantiation unit: mode FAITHFUL, d = 2, p + 1 = 2 (compiled with --fmad=false)
#include "../fdg_dispatch.cuh"

fdg::LaunchFn fdg_pick_faithful_d2_p2(int vf, bool curved, int logs)
{
    return fdg::pick_flux<2, 2, fdg::FAITHFUL>(vf, curved, logs);
}
