"""Device verification reductions (E/harness.py:165-179) against numpy /
hashlib on the same bytes."""
import hashlib

import numpy as np
import pytest
import torch

import paper_2106_15869_b200 as eik
from paper_2106_15869_b200.harness import field_digest

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def host_digest(b: bytes, chunk=1 << 16) -> str:
    return hashlib.sha256(b"".join(hashlib.sha256(b[o:o + chunk]).digest() for o in range(0, len(b), chunk))).hexdigest()


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_field_max_diff_device_equals_numpy(dtype):
    rng = np.random.default_rng(5)
    for n in (1, 31, 1000, 100_003):
        a = rng.random(n).astype(dtype)
        b = (a + rng.normal(0, 1e-3, n)).astype(dtype)
        k = rng.integers(0, n, max(1, n // 10))
        a[k], b[k] = np.inf, np.inf  # equal infinities count 0
        k2 = rng.integers(0, n, max(1, n // 20))
        a[k2], b[k2] = -np.inf, -np.inf
        want = eik.field_max_diff(a, b)
        got = eik.field_max_diff(torch.as_tensor(a, device=DEV), torch.as_tensor(b, device=DEV))
        assert got == want
    a = np.array([1.0, np.inf, 2.0], dtype=dtype)
    b = np.array([1.0, -np.inf, 2.5], dtype=dtype)  # opposite infinities: inf
    assert eik.field_max_diff(torch.as_tensor(a, device=DEV), torch.as_tensor(b, device=DEV)) == np.inf
    a[2] = np.nan
    assert np.isnan(eik.field_max_diff(torch.as_tensor(a, device=DEV), torch.as_tensor(b, device=DEV)))
    assert np.isnan(eik.field_max_diff(a, b))
    e = torch.empty(0, dtype=torch.float64, device=DEV)
    assert eik.field_max_diff(e, e) == 0.0
    with pytest.raises(ValueError):
        eik.field_max_diff(torch.zeros(3, dtype=torch.float64, device=DEV), torch.zeros(4, dtype=torch.float64, device=DEV))


def test_field_sha256_streams_a_device_field():
    rng = np.random.default_rng(6)
    for n in (0, 1, 1000, (1 << 26) // 8 * 3 + 17):  # > 2 staging pieces
        a = rng.random(n)
        assert eik.field_sha256(torch.as_tensor(a, device=DEV)) == hashlib.sha256(a.tobytes()).hexdigest()


def test_field_digest_device_equals_host():
    rng = np.random.default_rng(7)
    for nb in (0, 1, 55, 56, 63, 64, 65, 119, 120, 128, 65536, 65536 + 8, 3 * 65536 - 1, 1_000_003):
        b = rng.integers(0, 256, nb, dtype=np.uint8)
        t = torch.as_tensor(b, device=DEV)
        assert field_digest(t) == host_digest(b.tobytes()) == field_digest(b), nb
    for chunk in (64, 4096):
        b = rng.integers(0, 256, 10_000, dtype=np.uint8)
        assert field_digest(torch.as_tensor(b, device=DEV), chunk) == host_digest(b.tobytes(), chunk)
    a = rng.random((7, 9, 11))
    assert field_digest(torch.as_tensor(a, device=DEV)) == field_digest(a)
    # the piece hash itself is FIPS 180-4 SHA-256: one piece == hashlib
    b = rng.integers(0, 256, 1000, dtype=np.uint8)
    assert field_digest(torch.as_tensor(b, device=DEV), 1024) == hashlib.sha256(
        hashlib.sha256(b.tobytes()).digest()).hexdigest()


@pytest.mark.slow
def test_1024_cubed_checks_stay_on_the_device():
    """1024^3 float64 fields (8 GiB each): max diff and digest without a full D2H copy."""
    torch.cuda.empty_cache()
    n = 1024
    a = torch.rand((n, n, n), dtype=torch.float64, device=DEV)
    b = a.clone()
    v = b.view(-1)[123_456_789].item()
    b.view(-1)[123_456_789] = v + 0.5
    b.view(-1)[5] = np.inf
    a.view(-1)[5] = np.inf
    assert eik.field_max_diff(a, b) == abs((v + 0.5) - v)
    d1, d2 = field_digest(a), field_digest(b)
    b.view(-1)[123_456_789] = v
    assert d1 != d2 and field_digest(b) == d1
    del a, b
    torch.cuda.empty_cache()
