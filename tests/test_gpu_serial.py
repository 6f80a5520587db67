"""Serialisation at the boundary (versioned little-endian binary with magic,
params digest and per-prime residue arrays; keys sent once and cached).
The blob layout documented in include/mmfhe.h is parsed here by an independent reader
(struct.unpack + an FNV-1a written from its definition), so a layout change on one side
fails the test; loaded keys are checked by a relinearisation bit-exact with the oracle."""
import struct

import numpy as np
import pytest

from oracle import ckks as orc
from synth.params import toy

from gpu_util import ct_in, ct_out, make_ctx, residues

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def m(cuda_ctx_ok):
    from paper_2603_22437_b200 import build, mmfhe
    build.build()
    return mmfhe


def fnv1a64(data: bytes) -> int:
    h = 0xcbf29ce484222325
    for b in data:
        h ^= b
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def digest(P) -> int:
    b = b"mmfhe-params-v1" + struct.pack("<II", P.log_n, len(P.q)) + struct.pack(f"<{len(P.q)}Q", *P.q)
    b += struct.pack("<I", len(P.p)) + struct.pack(f"<{len(P.p)}Q", *P.p) + struct.pack("<I", P.alpha)
    return fnv1a64(b)


def parse(blob: bytes, n: int):
    assert blob[:8] == b"MMFHEBLB"
    (ver, kind, dig, log_n, level, npol, nsl, scale, step, nrows, pay) = struct.unpack_from("<IIQIIIIdiIQ", blob, 8)
    off = 64 + (nrows + 7) // 8 * 8
    primes = list(blob[64:64 + nrows])
    res = np.frombuffer(blob, dtype="<u8", count=nrows * n, offset=off).reshape(nrows, n)
    assert pay == nrows * n * 8 and len(blob) == off + pay
    return dict(version=ver, kind=kind, digest=dig, log_n=log_n, level=level, n_polys=npol, n_slots=nsl,
                scale=scale, step=step, primes=primes, res=res)


def test_ct_blob_layout_and_round_trip(m):
    import torch
    P = toy(log_n=10, n_q=4, scale_bits=40, n_p=2, alpha=2)
    keys = orc.keygen(P, seed=8101)
    ct = orc.encrypt_vector(P, keys, np.linspace(-1, 1, P.n // 2), 3, seed=8102, index=0)
    ctx = make_ctx(m, P)
    assert ctx.params_digest() == digest(P)
    blob = ctx.serialize_ct(ct_in(m, P, ct))
    h = parse(blob, P.n)
    assert (h["version"], h["kind"], h["digest"], h["log_n"], h["level"], h["n_polys"]) == (1, 0, digest(P), P.log_n,
                                                                                          3, 2)
    assert h["n_slots"] == P.n // 2 and h["scale"] == ct.scale and h["step"] == 0
    assert h["primes"] == [0, 1, 2, 3] * 2
    assert np.array_equal(h["res"], np.concatenate(ct.c))
    # host buffer in, the same blob; device buffer out
    assert ctx.serialize_ct(ct_in(m, P, ct, device=False)) == blob
    out = ct_out(m, P, 3)
    ctx.deserialize_ct(blob, out)
    assert np.array_equal(residues(out), np.stack(ct.c)) and out.scale == ct.scale and out.level == 3
    # an evaluation-form (NTT) device ciphertext serialises to the same coefficient-form blob
    x = ct_in(m, P, ct)
    ctx.ntt(x.data.view(-1, P.n), [i % 4 for i in range(8)])
    x.form = m.FORM_EVAL
    torch.cuda.synchronize()
    assert ctx.serialize_ct(x) == blob


def test_blob_errors_are_format_errors(m):
    P = toy(log_n=10, n_q=4, scale_bits=40, n_p=2, alpha=2)
    keys = orc.keygen(P, seed=8111)
    ct = orc.encrypt_vector(P, keys, np.ones(8), 3, seed=8112, index=0)
    ctx = make_ctx(m, P)
    blob = ctx.serialize_ct(ct_in(m, P, ct))
    bad = [b"XMFHEBLB" + blob[8:],                                   # magic
           blob[:8] + struct.pack("<I", 2) + blob[12:],              # version
           blob[:16] + struct.pack("<Q", digest(P) ^ 1) + blob[24:],  # params digest
           blob[:-8],                                                # truncated
           blob[:64] + bytes([5]) + blob[65:]]                       # prime order
    r = bytearray(blob)
    r[-8:] = struct.pack("<Q", P.q[3])                               # unreduced residue
    bad.append(bytes(r))
    for b in bad:
        with pytest.raises(m.MmfheError) as e:
            ctx.deserialize_ct(b, ct_out(m, P, 3))
        assert e.value.name == "E_FORMAT"
    # a ctx with other primes rejects the blob by digest
    P2 = toy(log_n=10, n_q=5, scale_bits=40, n_p=2, alpha=2)
    with pytest.raises(m.MmfheError) as e:
        make_ctx(m, P2).deserialize_ct(blob, ct_out(m, P2, 3))
    assert e.value.name == "E_FORMAT"


def test_serialized_keys_load_and_switch_bit_exact(m):
    """Relinearisation and Galois keys shipped as blobs (client packaging -> cloud load)
    give HMult and HRot residues equal to the oracle's."""
    P = toy(log_n=10, n_q=4, scale_bits=40, n_p=2, alpha=2)
    keys = orc.keygen(P, seed=8121, rotations=[3])
    a = orc.encrypt_vector(P, keys, np.linspace(-1, 1, P.n // 2), 3, seed=8122, index=0)
    ev = orc.Evaluator(P, keys.rlk, keys.gk)
    want_mul, want_rot = ev.mul_relin(a, a), ev.rotate(a, 3)
    packer = make_ctx(m, P)
    rl = packer.serialize_key(m.SER_RELIN_KEY, 0, keys.rlk)
    gk = packer.serialize_key(m.SER_GALOIS_KEY, 3, keys.gk[3])
    h = parse(gk, P.n)
    assert h["kind"] == 2 and h["step"] == 3 and h["n_polys"] == P.dnum() and h["n_slots"] == P.K
    assert np.array_equal(h["res"], keys.gk[3].reshape(-1, P.n))
    ctx = make_ctx(m, P)
    ctx.load_key_serialized(rl)
    ctx.load_key_serialized(gk)
    o = ct_out(m, P, 3)
    ctx.hmult(ct_in(m, P, a), ct_in(m, P, a), o)
    assert np.array_equal(residues(o), np.stack(want_mul.c))
    o = ct_out(m, P, 3)
    ctx.hrot(ct_in(m, P, a), 3, o)
    assert np.array_equal(residues(o), np.stack(want_rot.c))
    with pytest.raises(m.MmfheError) as e:
        ctx.load_key_serialized(packer.serialize_ct(ct_in(m, P, a)))
    assert e.value.name == "E_FORMAT"
