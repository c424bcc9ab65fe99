"""Host-side FIFO bookkeeping of the device reservoir ring (core.FeatureReservoir):
the write position and the (head, len) mirror that the graph-captured ring
append (xgs_vq_ring_write_dev) relies on, against a plain FIFO model of the
reference's FeatureReservoir.extend (core.py:178-203).  No GPU: only the
bookkeeping is exercised."""

import numpy as np

from paper_2603_09632_b200.core import FeatureReservoir


def _device_start(start, n, cap):
    """ring_advance_kernel: the device-side write position after appending n rows."""
    return 0 if n >= cap else (start + n) % cap


def test_account_matches_a_fifo_model_and_the_device_position():
    rng = np.random.default_rng(0)
    for cap in (1, 3, 8, 17):
        res = FeatureReservoir(cap, 4)
        fifo = []                      # row ids in FIFO order, last cap kept
        next_id = 0
        dev_start = res._write_pos()
        for _ in range(200):
            n = int(rng.choice([0, 1, 2, cap - 1 if cap > 1 else 1, cap, cap + 3, int(rng.integers(0, 3 * cap + 1))]))
            # where each appended row lands (physical ring row), as the device writes them
            phys = {}
            for j in range(n):
                if n >= cap:
                    if j >= n - cap:
                        phys[next_id + j] = j - (n - cap)
                else:
                    phys[next_id + j] = (dev_start + j) % cap
            res._account(n)
            dev_start = _device_start(dev_start, n, cap)
            fifo.extend(range(next_id, next_id + n))
            fifo = fifo[-cap:]
            next_id += n
            assert len(res) == len(fifo)
            assert res._write_pos() == dev_start
            # logical index i of the FIFO sits at physical row (head + i) % cap
            ring = {}
            for rid, p in phys.items():
                ring[p] = rid
            for i, rid in enumerate(fifo):
                if rid in phys:
                    assert (res._head + i) % cap == phys[rid]
