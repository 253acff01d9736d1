"""The paper's performance-index protocol on the device (
reference harness.measure_pid, harness.py:445-477).

PID = wall time of one RHS evaluation / #DOF, #DOF = (p+1)^d elements (every
volume node one DOF). Protocol: isentropic vortex (epsilon = 20) on
[-5, 5]^d, 8 elements per direction, Carpenter-Kennedy RK54 with the CFL
step size of the initial state (stable_dt, cfl 0.5), 90 steps = 450 RHS
evaluations, mean and std over 5 repeats from the initial state after one
warm-up evaluation.

Here every RK stage is ONE fused kernel (volume + interfaces + stage update,
DeviceStepper) and the 90 steps are captured once as a CUDA graph; each
repeat replays it between two CUDA events. ``measure_pid_device`` returns
the same fields as the reference's PidResult plus the device timing details.
"""

import statistics

import numpy as np


def build_pid_run(d=3, p=3, elements=8, mesh="cartesian", amplitude=0.1, volume_flux="ranocha",
                  surface_flux="ranocha", precompute="none", kernel="batched", ic="isentropic_vortex",
                  epsilon=20.0, gamma=1.4):
    """(setup, u0 host, RhsConfig) of one PID configuration (harness.build_run)."""
    from .discretization import RhsConfig, build_setup
    from .euler import GasParams
    from .geometry import build_mesh
    from .ics import DOMAIN_HI, DOMAIN_LO, initial_state
    from .operators import lgl_operator

    gas = GasParams(gamma)
    m = build_mesh((elements,) * d, bounds=(DOMAIN_LO, DOMAIN_HI), amplitude=amplitude if mesh == "curved" else 0.0)
    setup = build_setup(m, lgl_operator(p), gas)
    u0 = initial_state(ic, setup.coords, gas, epsilon=epsilon)
    cfg = RhsConfig(volume_flux=volume_flux, surface_flux=surface_flux, precompute=precompute, kernel=kernel)
    return setup, u0, cfg


def measure_pid_device(setup, u0, config, n_steps=90, repeats=5, cfl=0.5):
    """PID of the fused device stepper on (setup, u0, config)."""
    import torch

    from .device import device_mesh_for
    from .timeint import RK54, DeviceStepper, StepController, stable_dt

    dm = device_mesh_for(setup)
    st = DeviceStepper(dm, config, RK54)
    u_init = torch.as_tensor(np.ascontiguousarray(u0), device=dm.device)
    dt = stable_dt(u_init, None, setup.metrics, setup.gas, setup.op.degree, StepController(cfl), setup=setup)
    st.step(u_init, dt)  # warm-up (kernel attributes, occupancy), checked
    u_in = u_init.clone()  # static input buffer of the graph
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        u = u_in
        for _ in range(n_steps):
            u = st.step(u, dt, check=False)
    u_out = u
    dofs = setup.n_elements * setup.n_nodes
    samples = []
    for _ in range(repeats):
        u_in.copy_(u_init)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        graph.replay()
        b.record()
        b.synchronize()
        samples.append(a.elapsed_time(b) * 1e-3 / (5 * n_steps * dofs))
    final = u_out.cpu().numpy()
    if not np.all(np.isfinite(final)):
        from .errors import DivergenceError

        raise DivergenceError("non-finite state after the PID run")
    return {
        "mean_pid": statistics.mean(samples),
        "std_pid": statistics.pstdev(samples),
        "n_rhs": 5 * n_steps,
        "dofs": dofs,
        "dt": dt,
        "final": final,
        "how": "90 RK54 steps (450 fused stage kernels) captured in one CUDA graph, CUDA events around each replay",
    }
