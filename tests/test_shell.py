"""Host logic of the shell-only upload (pipeline_exec.write_core /
shell_boxes): the core is exactly the box every launch overwrites, and the
shell boxes tile the rest of the array without overlap.  CPU only."""
import itertools

import numpy as np
import pytest

from paper_2306_13002_b200 import pipeline_exec

# D3Q19 push targets (dz, dy, dx, q) of nests/d3q19.c (both arms)
D3Q19_C = [(0, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1), (1, 0, 0), (-1, 0, 0), (0, 1, 1), (0, 1, -1),
           (0, -1, 1), (0, -1, -1), (1, 1, 0), (-1, 1, 0), (1, -1, 0), (-1, -1, 0), (1, 0, 1), (-1, 0, 1),
           (1, 0, -1), (-1, 0, -1)]


class FakeKernel:
    def __init__(self, loop_of, targets, space):
        self.loop_of, self.targets, self.space = loop_of, targets, space

    def must_write(self, name):
        return list(self.loop_of) + [-1] * (8 - len(self.loop_of)), [tuple(t) + (0,) * (8 - len(t)) for t in self.targets]

    def iteration_space(self, scalars):
        return self.space


def covered(dims, boxes):
    m = np.zeros(dims, dtype=np.int32)
    for lo, hi in boxes:
        m[tuple(slice(a, b) for a, b in zip(lo, hi))] += 1
    return m


def test_d3q19_core_and_shell_tile_the_array():
    n = 10
    dims = (n, n, n, 19)
    k = FakeKernel([0, 1, 2, -1], [c + (q,) for q, c in enumerate(D3Q19_C)], [(1, n - 1)] * 3)
    core = pipeline_exec.write_core(k, "dst", dims, {})
    assert core == [(2, n - 2)] * 3 + [(0, 19)]
    shell = pipeline_exec.shell_boxes(dims, core)
    m = covered(dims, shell + [([c[0] for c in core], [c[1] for c in core])])
    assert (m == 1).all()        # disjoint and complete


def test_core_is_really_written():
    """Brute force: every core element is some point's store target."""
    n = 7
    dims = (n, n, n, 19)
    k = FakeKernel([0, 1, 2, -1], [c + (q,) for q, c in enumerate(D3Q19_C)], [(1, n - 1)] * 3)
    core = pipeline_exec.write_core(k, "dst", dims, {})
    written = np.zeros(dims, dtype=bool)
    for z, y, x in itertools.product(range(1, n - 1), repeat=3):
        for q, (dz, dy, dx) in enumerate(D3Q19_C):
            written[z + dz, y + dy, x + dx, q] = True
    sl = tuple(slice(a, b) for a, b in core)
    assert written[sl].all()


def test_missing_component_means_no_core():
    k = FakeKernel([0, 1, -1], [(0, 0, 0), (0, 0, 2)], [(0, 4), (0, 4)])
    assert pipeline_exec.write_core(k, "a", (4, 4, 3), {}) is None


def test_empty_space_and_shifted_core():
    k = FakeKernel([0, 1], [(0, 0)], [(3, 3), (0, 5)])
    assert pipeline_exec.write_core(k, "a", (8, 8), {}) is None
    k = FakeKernel([0, 1], [(1, -1)], [(0, 6), (1, 8)])
    assert pipeline_exec.write_core(k, "a", (8, 8), {}) == [(1, 7), (0, 7)]


@pytest.mark.parametrize("dims,core", [((5,), [(1, 3)]), ((6, 4), [(0, 6), (1, 3)]), ((3, 4, 5, 2), [(1, 2), (0, 4), (2, 5), (0, 2)])])
def test_shell_boxes_partition(dims, core):
    shell = pipeline_exec.shell_boxes(dims, core)
    m = covered(dims, shell + [([c[0] for c in core], [c[1] for c in core])])
    assert (m == 1).all()
