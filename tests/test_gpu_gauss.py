"""GPU parity of the Gauss-node family (the paper's second
scheme family -- zero-corner hybridized flux-differencing volume term with
entropy-projected face states, reference discretization.py:811-995,
batched.py:556-667).

Bars (written in each test):
* fdg_gauss_rhs given the oracle's projection and face traces: BITWISE equal
  to the C oracle (or_gauss_rhs, liboracle_cr), which is bitwise equal to
  the reference's scalar gauss path (tests/test_oracle.py);
* fdg_gauss_project against the numpy projection (the reference's own
  calls): <= 1e-14 relative to the largest face-state component (CUDA exp
  vs numpy exp, summation order of the boundary interpolation);
* the public rhs end to end against the reference's scalar and batched
  outputs: <= 1e-12 max(max|VOL_ref|, max|du_ref|) (cancellation-aware
  scale), the literal max-norm du error reported;
* the reference's error for an inadmissible projected face state.
"""

import numpy as np
import pytest

from oracle import oracle
from tests import golden_io as G

pytestmark = pytest.mark.gpu


def _P():
    import paper_2112_10517_b200 as P

    return P


def _combos(c, sname):
    for key in c:
        if not key.startswith("rhs_%s_" % sname):
            continue
        rest = key[len("rhs_%s_" % sname):]
        scheme = "gauss_surface_correction" if rest.startswith("gauss_surface_correction") else "gauss_fluxdiff"
        vf, sf = rest[len(scheme) + 1:].split("_")
        yield key, scheme, vf, sf


@pytest.mark.parametrize("name", G.GAUSS_CASES)
def test_gauss_rhs_kernel_bitwise_vs_oracle(name):
    import torch

    P = _P()
    from paper_2112_10517_b200.device import gauss_mesh_for, scheme_struct

    c = G.gauss_case(name)
    st = G.gauss_setup(name)
    d = st.d
    nrm = oracle.gauss_face_traces(st.metrics.ja, st.op, d)
    fnrm = np.stack([st.metrics.face_ja[n] for n in range(d)], axis=1)
    for sname in ("rand", "wave"):
        u = c["u_" + sname]
        proj = oracle.gauss_project(u, st.op)
        for key, scheme, vf, sf in _combos(c, sname):
            gm = gauss_mesh_for(st, scheme)
            dev = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")  # noqa: E731
            got = gm.rhs(dev(u), scheme_struct(vf, sf, "none", "reference"), proj=dev(proj), nrm=dev(nrm),
                         fnrm=dev(fnrm)).cpu().numpy()
            want = oracle.gauss_rhs(u, st, scheme, vf, sf, proj=proj, nrm=nrm, fnrm=fnrm, variant="cr")
            assert np.array_equal(got, want), key
            assert P is not None


@pytest.mark.parametrize("name", G.GAUSS_CASES)
def test_gauss_projection_kernel(name):
    import torch

    from paper_2112_10517_b200.device import gauss_mesh_for

    c = G.gauss_case(name)
    st = G.gauss_setup(name)
    gm = gauss_mesh_for(st, "gauss_fluxdiff")
    nrm_ref = oracle.gauss_face_traces(st.metrics.ja, st.op, st.d)
    for sname in ("rand", "wave"):
        u = c["u_" + sname]
        proj, nrm = gm.project(torch.as_tensor(u, device="cuda"))
        want = oracle.gauss_project(u, st.op)
        assert np.abs(proj.cpu().numpy() - want).max() <= 1e-14 * np.abs(want).max(), sname
        assert np.abs(nrm.cpu().numpy() - nrm_ref).max() <= 1e-15 * np.abs(nrm_ref).max(), sname


@pytest.mark.parametrize("name", G.GAUSS_CASES)
def test_gauss_rhs_public_api_vs_reference(name):
    P = _P()
    c = G.gauss_case(name)
    st = G.gauss_setup(name)
    for sname in ("rand", "wave"):
        u = c["u_" + sname]
        for key, scheme, vf, sf in _combos(c, sname):
            cnt = P.FluxCounter()
            got = P.rhs(u, st, P.RhsConfig(volume_scheme=scheme, volume_flux=vf, surface_flux=sf), counter=cnt)
            want = c[key]
            volkey = key.replace("rhs_", "vol_", 1)
            scale = max(np.abs(want).max(), np.abs(c[volkey]).max() if volkey in c else 0.0)
            err = np.abs(got - want).max()
            assert err <= 1e-12 * scale, (key, err / scale, err / np.abs(want).max())
            errb = np.abs(got - c[key.replace("rhs_", "rhsb_", 1)]).max()
            assert errb <= 1e-12 * scale, (key, errb / scale)
            assert (cnt.two_point_evals, cnt.one_point_evals, cnt.logmean_evals) == tuple(
                int(x) for x in c[key.replace("rhs_", "counts_", 1)]), key


def test_gauss_own_setup_and_errors():
    """This package's own Gauss setup (build_setup on gauss_operator) against
    the oracle on the same setup, and the reference's two error messages."""
    P = _P()
    gas = P.GasParams(1.4)
    setup = P.build_setup(P.build_mesh((3, 2, 2), bounds=(-1.0, 1.0), amplitude=0.08), P.gauss_operator(2), gas)
    rng = np.random.default_rng(4)
    q = np.empty((setup.n_elements, setup.n_nodes, 5))
    q[..., 0] = 1.0 + 0.3 * rng.random(q.shape[:2])
    q[..., 1:4] = 0.2 * (rng.random(q.shape[:2] + (3,)) - 0.5)
    q[..., 4] = 1.0 + 0.3 * rng.random(q.shape[:2])
    u = P.prim2cons(q, gas)
    cfg = P.RhsConfig(volume_scheme="gauss_fluxdiff", volume_flux="ranocha", surface_flux="llf")
    got = P.rhs(u, setup, cfg)
    want = oracle.gauss_rhs(u, setup, "gauss_fluxdiff", "ranocha", "llf")
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
    with pytest.raises(P.ConfigurationError, match="requires gauss operators"):
        P.rhs(u, P.build_setup(P.build_mesh((2, 2, 2), bounds=(-1.0, 1.0)), P.lgl_operator(2), gas), cfg)
    bad = u.copy()
    bad[1, 4, 0] = -1.0
    with pytest.raises(P.AdmissibilityError, match="element 1, node 4"):
        P.rhs(bad, setup, cfg)
    # admissible nodes whose extrapolated -w_last goes negative at a face
    # (Gauss boundary rows extrapolate with negative weights)
    q2 = q.copy()
    q2[0, :, 0] = 0.05
    q2[0, :, 4] = 50.0
    line = [0 * 9 + 1 * 3 + 0, 1 * 9 + 1 * 3 + 0, 2 * 9 + 1 * 3 + 0]  # direction-0 line through (., 1, 0)
    q2[0, line[1], 0], q2[0, line[1], 4] = 50.0, 0.05
    with pytest.raises(P.AdmissibilityError, match="entropy projection produced an inadmissible face state"):
        P.rhs(P.prim2cons(q2, gas), setup, cfg)
