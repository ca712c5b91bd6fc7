"""The five BASELINE.json workloads (workloads.py at the repository root) drawn from the
library's own Rng stream (pwb_rng_uniform, the reference's xorshift64*, util.hpp:83-98).
Test / bench convenience; nothing on the compute path imports it."""
from __future__ import annotations

from functools import partial
from typing import Optional

import workloads
from workloads import CONFIGS, Config, Inputs, neutralize  # noqa: F401

from . import rng_uniform


def generate(name: str, n_src: Optional[int] = None) -> Inputs:
    return workloads.generate(name, n_src, rng=rng_uniform)


normals = partial(workloads.normals, rng_uniform)
uniform_points = partial(workloads.uniform_points, rng_uniform)
clustered_points = partial(workloads.clustered_points, rng_uniform)
