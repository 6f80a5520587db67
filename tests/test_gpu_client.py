"""The trusted client on the GPU (include/mmfhe.h mmfhe_client_*): key
generation and encryption bit-identical to the oracle client (oracle.ckks.keygen / encrypt,
the same counter-based SplitMix64 streams of synth/prng.py), and their timing at PS4."""
import numpy as np
import pytest

from oracle import ckks as orc
from synth.params import toy

from gpu_util import ct_out, residues

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def m(cuda_ctx_ok):
    from paper_2603_22437_b200 import build, mmfhe
    build.build()
    return mmfhe


@pytest.mark.parametrize("alpha,n_p", [(2, 2), (1, 1)])
def test_client_keygen_matches_oracle(m, alpha, n_p):
    P = toy(log_n=10, n_q=5, scale_bits=40, n_p=n_p, alpha=alpha)
    # rotations, the conjugation (R28) and the conjugate-product key (R32)
    steps = [1, 3, P.n // 2 - 5, orc.CONJ, orc.CONJ_PROD]
    keys = orc.keygen(P, seed=8201, rotations=steps)
    ctx = m.Context.from_params(P)
    pk, rlk, gk = ctx.client_keygen(8201, steps)
    assert np.array_equal(pk, np.stack(keys.pk))
    assert np.array_equal(rlk, keys.rlk)
    for i, k in enumerate(steps):
        assert np.array_equal(gk[i], keys.gk[orc.key_id(P, k)]), k


def test_client_encrypt_matches_oracle_and_decrypts(m):
    P = toy(log_n=10, n_q=5, scale_bits=40, n_p=2, alpha=2)
    keys = orc.keygen(P, seed=8211)
    ctx = m.Context.from_params(P)
    rng = np.random.default_rng(3)
    vals = [rng.uniform(-1, 1, P.n // 2) for _ in range(5)]
    scale = float(2 ** P.scale_bits)
    lvl = 3
    pts = [m.Ct(np.ascontiguousarray(orc.encode(P, v, scale, lvl)), lvl, scale, P.n // 2, P.log_n, m.FORM_COEFF, 1)
           for v in vals]
    outs = [ct_out(m, P, lvl) for _ in vals]
    ctx.client_encrypt(np.ascontiguousarray(np.stack(keys.pk)), pts, 8212, 7, outs)
    for i, (v, o) in enumerate(zip(vals, outs)):
        want = orc.encrypt(P, keys, pts[i].data, lvl, scale, P.n // 2, seed=8212, index=7 + i)
        assert np.array_equal(residues(o), np.stack(want.c))
        assert o.level == lvl and o.scale == scale
        got = orc.decrypt_vector(P, keys, orc.Ct([residues(o)[0], residues(o)[1]], lvl, scale, P.n // 2))
        assert np.max(np.abs(got - v)) < 1e-6
