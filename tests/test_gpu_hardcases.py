"""The hardest-to-round binary32 inputs of every function (tests/golden/
hardcases/, found by the GPU screen over all 2^32 inputs and ranked by the
oracle's MPFR boundary distance) through the full kernels, all four modes."""
import os

import numpy as np
import pytest

import paper_2605_15547_b200 as crvec

pytestmark = pytest.mark.gpu
DIR = os.path.join(os.path.dirname(__file__), "golden", "hardcases")


def load(name):
    p = os.path.join(DIR, name + ".txt")
    if not os.path.exists(p):
        pytest.fail(f"missing corpus {p} (python tools/hard_cases.py {name})")
    rows = [l.split() for l in open(p) if l.strip() and not l.startswith("#")]
    x = np.array([int(r[0], 16) for r in rows], np.uint32)
    want = np.array([[int(v, 16) for v in r[3:7]] for r in rows], np.uint32)
    return x, want


@pytest.mark.parametrize("name", crvec.F32_FUNCS)
def test_hardest_cases_all_modes(cuda, name):
    x, want = load(name)
    assert len(x) > 0
    # embed each hard input among random co-resident lanes (SPEC corpus_check)
    rng = np.random.default_rng(1)
    pad = rng.uniform(-2, 2, 1023 * len(x)).astype(np.float32).view(np.uint32)
    xx = np.concatenate([x, pad])
    perm = rng.permutation(len(xx))
    xs = xx[perm]
    pos = np.argsort(perm)[: len(x)]
    t = cuda.from_numpy(xs.view(np.float32)).cuda()
    for m in range(4):
        got = crvec.eval_f32(name, t, m).cpu().numpy().view(np.uint32)[pos]
        bad = np.nonzero(got != want[:, m])[0]
        assert len(bad) == 0, (name, m, [hex(int(x[i])) for i in bad[:5]])
