// instantiation unit: mode FAST, d = 2, p + 1 = 4
#include "../fdg_dispatch.cuh"

fdg::LaunchFn fdg_pick_fast_d2_p4(int vf, bool curved, int logs)
{
    return fdg::pick_flux<2, 4, fdg::FAST>(vf, curved, logs);
}
