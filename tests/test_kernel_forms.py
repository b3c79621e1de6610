"""The A/B kernel forms stay parity-green: the production step uses tcgen05
for the coarse no-grad SDF, the taped forward and both backward kernels
(gsb_step.cuh: GSB_T5=2, GSB_T5_FWD=4, GSB_T5_BWD=1, GSB_T5_COL=1).  The alternatives
(mma.sync everywhere; tcgen05 everywhere, the importance-pass SDF included; the
taped forward at 3 CTAs per SM, and with the finest level's corners staged in
shared memory by cp.async) are read
once per process from the environment, so each runs the float step parity
tests of test_gpu_step.py and the conditioned float32 parity of
test_f32_parity.py in a child process against the same oracle goldens."""

import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))

FORMS = {
    "mma_sync": {"GSB_T5": "0", "GSB_T5_FWD": "0", "GSB_T5_BWD": "0", "GSB_T5_COL": "0"},
    "tcgen05_all": {"GSB_T5": "1", "GSB_T5_FWD": "4", "GSB_T5_BWD": "1", "GSB_T5_COL": "1"},
    "fwd_3cta": {"GSB_T5_FWD": "3"},
    "fwd_staged": {"GSB_T5_FWD": "5"},
}


@pytest.mark.gpu
@pytest.mark.parametrize("form", sorted(FORMS))
def test_alternative_kernel_forms_match_reference(form):
    env = dict(os.environ, **FORMS[form])
    base = [sys.executable, "-m", "pytest", "-m", "gpu", "-q", "-x", "-p", "no:cacheprovider"]
    for cmd in (base + [os.path.join(HERE, "test_gpu_step.py"), "-k",
                        "step_ or deterministic or two_iterations"],
                base + [os.path.join(HERE, "test_f32_parity.py")]):  # conditioned 1e-4 / 1e-5
        r = subprocess.run(cmd, env=env, cwd=os.path.dirname(HERE), capture_output=True, text=True,
                           timeout=900)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
        assert " passed" in r.stdout
