"""hgrd_gpu_buffer_write_async (the B200-side upload that overlaps the next
batch's H2D copy with the current check): the next check / read / write of
the buffer waits for the copy on the device, so results are those of the
synchronous write.  Expected reports: programs.histogram_pow2_expected,
pinned to the reference by test_oracle_pin.test_structural_predictors_pinned."""
import numpy as np
import pytest

import paper_2604_02106_b200 as hg
import programs

pytestmark = pytest.mark.gpu


def _pinned(a):
    import torch
    t = torch.empty(a.size, dtype=torch.int64, pin_memory=True).numpy()
    t[:] = a
    return t


def test_write_async_then_read(gpu):
    gpu.reset()
    n = 1 << 22
    h = gpu.alloc(n)
    src = _pinned(np.arange(n, dtype=np.int64) * 7 - 3)
    gpu.write_async(h, src)
    out = np.empty(n, dtype=np.int64)
    gpu.read(h, out)
    assert np.array_equal(out, src)
    # partial upload over a zero-initialised buffer (zeroing ordered first)
    h2 = gpu.alloc(n)
    gpu.write_async(h2, src[:1000], 5)
    gpu.read(h2, out)
    assert not out[:5].any() and np.array_equal(out[5:1005], src[:1000]) and not out[1005:].any()


@pytest.mark.parametrize("update", ["store", "atomic_block"])
def test_pipelined_histogram(gpu, update):
    """Two buffer sets, step k+1's data uploaded while step k is checked;
    the sets hold different data (seeds), so a check that ran before its
    upload landed would report the other seed's races."""
    n, bins = 1 << 22, 1 << 16
    gpu.reset()
    low = hg.lower(programs.histogram(n, bins, update, host_init=False), "h")
    sets = []
    for seed in (programs.HIST_SEED, programs.HIST_SEED + 1):
        h = {"data": gpu.alloc(n), "hist": gpu.alloc(bins)}
        host = _pinned(programs.histogram_data(n, bins, seed))
        spec = hg.LaunchSpec(low, (n // 256, 1, 1), (256, 1, 1), 32, handles=h)
        sets.append((h, host, spec, programs.histogram_pow2_expected(n, bins, update, seed)))
    assert sets[0][3] != sets[1][3]
    gpu.write_async(sets[0][0]["data"], sets[0][1])
    steps = 6
    for k in range(steps):
        if k + 1 < steps:
            nxt = sets[(k + 1) % 2]
            gpu.write_async(nxt[0]["data"], nxt[1])
        _, _, spec, want = sets[k % 2]
        got = gpu.check_launch(spec)
        assert [(r["kind"], r["address"], r["threadA"], r["threadB"])
                for r in got["races"]] == want, k
