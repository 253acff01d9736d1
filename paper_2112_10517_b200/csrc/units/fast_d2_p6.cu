// instantiation unit: mode FAST, d = 2, p + 1 = 6
#include "../fdg_dispatch.cuh"

fdg::LaunchFn fdg_pick_fast_d2_p6(int vf, bool curved, int logs)
{
    return fdg::pick_flux<2, 6, fdg::FAST>(vf, curved, logs);
}
