"""mt19937_64 (the published Matsumoto-Nishimura 64-bit Mersenne Twister, the
engine std::mt19937_64 names) for host-side seeding that must reproduce the
reference's KruskalModel::random stream (cp_als.cpp:87-99). Pure Python:
only used for small factor initialisation."""

_N, _M = 312, 156
_UPPER, _LOWER = 0xFFFFFFFF80000000, 0x7FFFFFFF
_MASK = (1 << 64) - 1


class mt19937_64:
    def __init__(self, seed: int):
        mt = [0] * _N
        mt[0] = seed & _MASK
        for i in range(1, _N):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _MASK
        self.mt = mt
        self.idx = _N

    def _twist(self):
        mt = self.mt
        for i in range(_N):
            y = (mt[i] & _UPPER) | (mt[(i + 1) % _N] & _LOWER)
            v = mt[(i + _M) % _N] ^ (y >> 1)
            if y & 1:
                v ^= 0xB5026F5AA96619E9
            mt[i] = v
        self.idx = 0

    def next(self) -> int:
        if self.idx >= _N:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000 & _MASK
        y ^= (y << 37) & 0xFFF7EEE000000000 & _MASK
        y ^= y >> 43
        return y & _MASK
