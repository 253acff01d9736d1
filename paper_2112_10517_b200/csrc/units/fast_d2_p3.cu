// instantiation unit: mode FAST, d = 2, p + 1 = 3
#include "../fdg_dispatch.cuh"

fdg::LaunchFn fdg_pick_fast_d2_p3(int vf, bool curved, int logs)
{
    return fdg::pick_flux<2, 3, fdg::FAST>(vf, curved, logs);
}
