"""CPU check of the LRU replay helper used by the row-cache counter tests."""
import numpy as np

from tests.helpers.lru import lru_replay


def test_lru_replay_is_textbook_lru_when_no_pair_conflict():
    """The replay equals a plain LRU over the access sequence u, l, u, l, ... whenever the
    'not the other row' rule never fires (large capacity)."""
    import collections
    rng = np.random.default_rng(3)
    tr = rng.integers(0, 40, size=(500, 2))
    tr[tr[:, 0] == tr[:, 1], 1] += 1
    cache = collections.OrderedDict()
    h = 0
    for u, l in tr:
        for i in (int(u), int(l)):
            if i in cache:
                h += 1
                cache.move_to_end(i)
            else:
                cache[i] = 1
                if len(cache) > 64:
                    cache.popitem(last=False)
    assert lru_replay(tr, 64)[0] == h
