"""Pin the CPU oracle against the reference's own outputs (tests/golden)."""

import numpy as np
import pytest

from _golden import load, oracle_params, rel_maxnorm
from oracle import gridsurf_oracle as O

CASES = [(c, p) for c in ("tiny", "small") for p in ("double", "single")]
# gradients: max-abs-diff / max|g| per tensor
GRAD_TOL = {"double": 1e-9, "single": 1e-4}


@pytest.fixture(scope="module", params=CASES, ids=lambda cp: f"{cp[0]}-{cp[1]}")
def run(request):
    G = load(*request.param)
    P = oracle_params(G)
    it = G.meta["iteration"]
    batch = O.draw_ray_batch(G.ds, O.substream(G.cfg.seed, O.RAYS, it), G.cfg.batch_rays,
                             near=G.cfg.near, far=G.cfg.max_depth)
    R = O.train_objective(P, G.ds, batch, it, G.cfg)
    return G, P, batch, R


def test_init_params_bit_exact(run):
    G, P, _, _ = run
    for n, a in zip(P.names(), P.arrays()):
        np.testing.assert_array_equal(a, G.a[f"init_{n}"], err_msg=n)
        assert a.dtype == G.a[f"init_{n}"].dtype


def test_ray_batch_bit_exact(run):
    G, _, batch, _ = run
    for k in ("frame_ids", "pixels", "color", "depth_ray", "valid", "dir_cam"):
        np.testing.assert_array_equal(getattr(batch, k), G.a[f"batch_{k}"], err_msg=k)


def test_importance_rounds_bit_exact(run):
    G, _, _, R = run
    assert len(R["rounds"]) == G.cfg.importance_rounds
    for i, rd in enumerate(R["rounds"]):
        np.testing.assert_array_equal(rd["weights"], G.a[f"round{i}_weights"])
        np.testing.assert_array_equal(rd["depths"], G.a[f"round{i}_depths"])
        np.testing.assert_array_equal(rd["src"], G.a[f"round{i}_src"])
    np.testing.assert_array_equal(R["depths"], G.a["depths"])
    assert R["depths"].shape[1] == G.cfg.coarse_samples + \
        G.cfg.importance_rounds * G.cfg.importance_add


def test_render_weights_bit_exact(run):
    G, _, _, R = run
    np.testing.assert_array_equal(R["weights"], G.a["weights"])


def test_parts_and_extras(run):
    G, _, _, R = run
    for k, v in G.meta["parts"].items():
        if G.cfg.precision == "single" and k == "smooth":
            # grad-phi differs from numba's _nb_dx_forward by <= 1 ulp in
            # float32; the smoothness term is a difference of nearby
            # gradients, which amplifies that.
            assert R["parts"][k] == pytest.approx(v, rel=1e-5), k
            continue
        assert R["parts"][k] == v, (k, R["parts"][k], v)
    for k, v in G.meta["extras"].items():
        assert R["extras"][k] == v, k


def test_gradients_match_reference_tape(run):
    G, P, _, R = run
    tol = GRAD_TOL[G.cfg.precision]
    for n in P.names():
        g = R["grads"][n]
        ref = G.a[f"grad_{n}"]
        assert g.shape == ref.shape and g.dtype == ref.dtype, n
        assert rel_maxnorm(g, ref) <= tol, (n, rel_maxnorm(g, ref))


def test_adam_bit_exact_given_reference_grads(run):
    G, P, _, _ = run
    P1 = P.copy()
    names = P1.names()
    opt = O.Adam(P1.arrays(), P1.lrs())
    opt.step(P1.arrays(), [G.a[f"grad_{n}"] for n in names])
    for i, n in enumerate(names):
        np.testing.assert_array_equal(P1.arrays()[i], G.a[f"step1_{n}"], err_msg=n)
        np.testing.assert_array_equal(opt.m[i], G.a[f"step1_m_{n}"], err_msg=n)
        np.testing.assert_array_equal(opt.v[i], G.a[f"step1_v_{n}"], err_msg=n)


def test_two_iterations_double(run):
    G, P, _, _ = run
    if G.cfg.precision != "double":
        pytest.skip("post-Adam params are sign-sensitive for |g| ~ eps in single")
    P1 = P.copy()
    opt = O.Adam(P1.arrays(), P1.lrs())
    it = G.meta["iteration"]
    for k in (it, it + 1):
        R = O.train_step(P1, opt, G.ds, G.cfg, k)
    for k, v in G.meta["parts1"].items():
        assert R["parts"][k] == pytest.approx(v, rel=1e-9, abs=1e-14), k
    for i, n in enumerate(P1.names()):
        assert rel_maxnorm(P1.arrays()[i], G.a[f"final_{n}"]) <= 1e-8, n


def test_relu_flips_ratio_semantics():
    """The oracle's alpha-ratio kink switch (relu_flips["ratio"], used by
    tests/test_f32_parity.py): flipping the branch of min(ratio, 1) at one
    interval leaves every value and loss part unchanged and changes the
    gradients only through that interval's two samples."""
    G = load("tiny", "double")
    P = oracle_params(G)
    it = G.meta["iteration"]
    batch = O.draw_ray_batch(G.ds, O.substream(G.cfg.seed, O.RAYS, it), G.cfg.batch_rays,
                             near=G.cfg.near, far=G.cfg.max_depth)
    R0 = O.train_objective(P, G.ds, batch, it, G.cfg)
    # the interval with the largest phi_bar jump if flipped
    row, j = np.unravel_index(np.argmax(R0["ratio_jump"]), R0["ratio_jump"].shape)
    R1 = O.train_objective(P, G.ds, batch, it, G.cfg, relu_flips={"ratio": [(int(row), int(j))]})
    assert R1["parts"] == R0["parts"]
    np.testing.assert_array_equal(R1["phi"], R0["phi"])
    assert any(not np.array_equal(R1["grads"][n], R0["grads"][n]) for n in R0["grads"])
    # and flipping it back is the identity
    R2 = O.train_objective(P, G.ds, batch, it, G.cfg,
                           relu_flips={"ratio": [(int(row), int(j)), (int(row), int(j))]})
    for n in R0["grads"]:
        np.testing.assert_array_equal(R2["grads"][n], R0["grads"][n])
