// instantiation unit: mode FAST, d = 3, p + 1 = 2
#include "../fdg_dispatch.cuh"

fdg::LaunchFn fdg_pick_fast_d3_p2(int vf, bool curved, int logs)
{
    return fdg::pick_flux<3, 2, fdg::FAST>(vf, curved, logs);
}
