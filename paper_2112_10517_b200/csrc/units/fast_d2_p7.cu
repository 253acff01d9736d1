// instantiation unit: mode FAST, d = 2, p + 1 = 7
#include "../fdg_dispatch.cuh"

fdg::LaunchFn fdg_pick_fast_d2_p7(int vf, bool curved, int logs)
{
    return fdg::pick_flux<2, 7, fdg::FAST>(vf, curved, logs);
}
