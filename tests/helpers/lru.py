"""Replay of the row cache's replacement policy on a pair trajectory (test helper)."""
import collections


def lru_replay(trace, slots):
    """The row cache's replacement policy (smo_kernel.cuh), replayed on a
    pair trajectory: per step look up u and l; a missing row takes the least recently
    used slot -- never the slot holding the other row of the pair -- and each row's slot
    becomes the most recently used (u first, then l).  Returns (hits, misses)."""
    order = collections.OrderedDict((s, None) for s in range(slots - 1, -1, -1))  # last = most recent
    owner = [-1] * slots
    where = {}
    hits = misses = 0

    def victim(avoid):
        it = iter(order)
        v = next(it)
        if v == avoid:
            v = next(it)
        if owner[v] >= 0:
            del where[owner[v]]
        return v

    for u, l in trace:
        su, sl = where.get(int(u), -1), where.get(int(l), -1)
        hits += (su >= 0) + (sl >= 0)
        misses += (su < 0) + (sl < 0)
        if su < 0:
            su = victim(sl)
            owner[su] = int(u); where[int(u)] = su
        order.move_to_end(su)
        if sl < 0:
            sl = victim(su)
            owner[sl] = int(l); where[int(l)] = sl
        order.move_to_end(sl)
    return hits, misses
