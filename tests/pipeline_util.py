"""Run the PRODUCT preprocessing pipeline step by step (the reference's
tests/helpers.py:117-125 shape) and collect its parity arrays."""

from __future__ import annotations

import numpy as np

import paper_2204_06666_b200 as E


def product_pipeline(n, rows, cols, vals, tau, profile, assignment=None, n_parts_hint=None,
                     seed=0, rebalance=False):
    m = E.CooMatrix(n, n, rows, cols, vals)
    prof = E.DeviceProfile(*profile) if not isinstance(profile, E.DeviceProfile) else profile
    params = E.compute_params(n, tau, prof)
    g = E.build_graph(m)
    if assignment is None:
        parts = E.partition_graph(g, params.n_parts, params.vec_cache_size, seed=seed)
    elif rebalance:
        parts = E.PartitionMap.from_assignment(assignment, n_parts=n_parts_hint)
        if parts.n_parts < params.n_parts:
            parts = E.PartitionMap.from_assignment(parts.assignment, n_parts=params.n_parts)
        if int(parts.part_sizes.max(initial=0)) > params.vec_cache_size:
            parts = E.rebalance_partition(g, parts, params.vec_cache_size)
    else:
        parts = E.PartitionMap.from_assignment(assignment, n_parts=n_parts_hint)
    cls = E.classify_rows(m, parts)
    plan = E.build_reorder_plan(cls, params, parts)
    e = E.assemble_ehyb(m, plan, params, parts)
    return m, params, g, parts, cls, plan, e
