"""Oracle: the count-sketch hash pair (h, s) — PAPER.md §3.1 P:L200-204 ("two pair-wise
independent hash functions h: [d]->[k] and s: [d]->{-1,+1} ... their selection from the
families H and S is random").  The paper gives no construction; our reading (DESIGN.md §3,
reading 2; SURVEY §8(c) "Documented hash") is the Carter–Wegman 2-universal family over the
Mersenne prime p = 2^61-1, keyed by the stream *id* so add/delete never move other streams
(S:L271, L288), with its random parameters drawn from splitmix64 (Steele, Lea, Flood 2014)
seeded by the sketch seed.  Pure Python integers: exact, no shared code with the C++ hash.

Test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations

P61 = (1 << 61) - 1
_MASK = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15


def splitmix64_stream(seed: int, count: int) -> list[int]:
    """`count` successive splitmix64 outputs starting from state = seed (all mod 2^64)."""
    state = seed & _MASK
    out = []
    for _ in range(count):
        state = (state + _GAMMA) & _MASK
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        out.append(z ^ (z >> 31))
    return out


def cw_params(seed: int) -> tuple[int, int, int, int]:
    """(a, b, c, e): successive splitmix64 outputs reduced mod p; zero a or c is redrawn."""
    state = seed & _MASK
    vals = []

    def nxt():
        nonlocal state
        state = (state + _GAMMA) & _MASK
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        return (z ^ (z >> 31)) % P61

    a = nxt()
    while a == 0:
        a = nxt()
    b = nxt()
    c = nxt()
    while c == 0:
        c = nxt()
    e = nxt()
    vals = (a, b, c, e)
    return vals


def plan_count_sketch(ids, k: int, seed: int) -> tuple[list[int], list[int]]:
    """For each stream id: group h(id) = ((a x + b) mod p) mod k and sign s(id) = +1 if
    ((c x + e) mod p) is even else -1, with x = id mod p."""
    a, b, c, e = cw_params(seed)
    groups, signs = [], []
    for i in ids:
        x = int(i) % P61
        groups.append(((a * x + b) % P61) % k)
        signs.append(1 if ((c * x + e) % P61) % 2 == 0 else -1)
    return groups, signs
