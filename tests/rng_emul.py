"""Pure-Python emulation of the reference SeededRng stream
(proj/include/adagio/rng.hpp:49-91) for driving the reference test
generators (TEST INFRASTRUCTURE).  Checked against the compiled reference in
tests/golden/rng_golden.json by tests/test_oracle.py."""
import math

M64 = (1 << 64) - 1
GOLDEN = 0x9e3779b97f4a7c15


class Stream:
    def __init__(self, seed):
        self.state = seed & M64
        self.cached = None

    def next_u64(self):
        self.state = (self.state + GOLDEN) & M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & M64
        z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & M64
        return z ^ (z >> 31)

    def below(self, bound):
        limit = (bound * (M64 // bound)) & M64
        v = self.next_u64()
        while v >= limit:
            v = self.next_u64()
        return v % bound

    def unit(self):
        return (self.next_u64() >> 11) * 2.0 ** -53

    def normal(self):
        if self.cached is not None:
            c, self.cached = self.cached, None
            return c
        u1 = self.unit()
        while u1 <= 0.0:
            u1 = self.unit()
        u2 = self.unit()
        radius = math.sqrt(-2.0 * math.log(u1))
        angle = 6.283185307179586476925286766559 * u2
        self.cached = radius * math.sin(angle)
        return radius * math.cos(angle)
