"""Pins of the shared input generator (synth/): published SplitMix64 vectors, value range, exactness."""
import numpy as np

from synth import SEED, gen_bits, gen_bits_at, gen_f32, splitmix64


def test_splitmix64_published_vectors():
    # Vigna's SplitMix64 reference: state 0 -> first output 0xE220A8397B1DCDAF.
    assert int(splitmix64(np.uint64(0))) == 0xE220A8397B1DCDAF
    # seed 1234567: the first five outputs of the reference generator (state advances by gamma).
    gamma = 0x9E3779B97F4A7C15
    expect = [6457827717110365317, 3203168211198807973, 9817491932198370423,
              4593380528125082431, 16408922859458223821]
    got = [int(splitmix64(np.uint64((1234567 + i * gamma) & (2**64 - 1)))) for i in range(5)]
    assert got == expect


def test_values_exact_and_in_range():
    w = gen_f32(SEED, 1, 3, 0, 1 << 16).astype(np.float64)
    assert np.all(np.abs(w) < 2.0 ** -7)
    m = w * 2.0 ** 30
    assert np.all(m == np.round(m))            # exactly m * 2^-30 with integer m
    assert np.all((m >= -(2 ** 23)) & (m < 2 ** 23))


def test_definition_by_hand():
    # element 5 of tensor 7 at version 2, recomputed with Python integers
    M = 2 ** 64 - 1
    key = (SEED ^ ((2 * 0x9E3779B97F4A7C15) & M) ^ (7 << 44) ^ 5) & M
    z = (key + 0x9E3779B97F4A7C15) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    x = z ^ (z >> 31)
    m = (x >> 40) - (1 << 23)
    want = np.float32(m * 2.0 ** -30).view(np.uint32)
    assert gen_bits(SEED, 2, 7, 5, 1)[0] == want


def test_versions_differ_and_index_forms_agree():
    a = gen_bits(SEED, 1, 0, 100, 4096)
    b = gen_bits(SEED, 2, 0, 100, 4096)
    assert np.mean(a != b) > 0.99
    idx = np.array([100, 4195, 1000, 101], dtype=np.uint64)
    assert np.array_equal(gen_bits_at(SEED, 1, 0, idx), a[(idx - 100).astype(np.int64)])


def test_specials_appear():
    bits = gen_bits(SEED, 1, 0, 0, 1 << 20, specials=True)
    assert np.count_nonzero(np.isnan(bits.view(np.float32))) > 0
    assert np.count_nonzero(bits == 0x7F7F8000) > 0
