"""CPU model of the mixed-radix Stockham passes in csrc/gfft.cu (general plane
sides): the same factorisation (8s, then 4s, then primes), stage index map
(butterfly j reads j + r N/R, writes (j // Ns) Ns R + j % Ns + q Ns) and
combined twiddle W_N^(r (j % Ns + q Ns) N / (Ns R)), checked against numpy's
FFT for the radices the kernels meet (2, 3, 4, 5, 7, 8, larger primes).  The CUDA
kernels themselves are checked on the GPU by tests/test_gpu_general_sizes.py."""
import numpy as np
import pytest


def factor(n):
    f = []
    while n % 8 == 0 and n > 8:
        f.append(8)
        n //= 8
    while n % 4 == 0 and n > 4:
        f.append(4)
        n //= 4
    p = 2
    while n > 1:
        while n % p == 0:
            f.append(p)
            n //= p
        p += 1
    return f


def stockham(x, inverse=False):
    N = len(x)
    W = np.exp(-2j * np.pi * np.arange(N) / N)
    if inverse:
        W = np.conj(W)
    src, dst, Ns = x.astype(np.complex128).copy(), np.zeros(N, np.complex128), 1
    for R in factor(N):
        M, step = N // R, N // (Ns * R)
        j = np.arange(M)
        jm, base = j % Ns, (j // Ns) * Ns * R + j % Ns
        for q in range(R):
            e = (jm + q * Ns) * step
            dst[base + q * Ns] = sum(src[j + r * M] * W[(r * e) % N] for r in range(R))
        src, dst = dst, src
        Ns *= R
    return src


@pytest.mark.parametrize("n", [8, 12, 30, 64, 96, 100, 125, 210, 1000, 1021, 1080, 1280, 1536, 134, 61 * 2])
def test_stockham_model_matches_numpy(n):
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    assert np.allclose(stockham(x), np.fft.fft(x), atol=1e-9 * n)
    assert np.allclose(stockham(x, inverse=True), np.fft.ifft(x) * n, atol=1e-9 * n)


def test_factorisation_products():
    for n in range(8, 4097, 37):
        f = factor(n)
        assert int(np.prod(f)) == n
        assert f == sorted(f, key=lambda r: (r not in (8, 4), r != 8))  # 8s, 4s, then the rest
