"""doctest::Approx semantics, so transcribed reference assertions keep their meaning.

doctest compares |a - b| < eps * (scale + max(|a|, |b|)) with scale = 1 and a
default eps of float epsilon * 100 (doctest.h, Approx::operator==).
"""


def approx_eq(a, b, eps=1.1920928955078125e-07 * 100, scale=1.0):
    a, b = float(a), float(b)
    return abs(a - b) < eps * (scale + max(abs(a), abs(b)))
