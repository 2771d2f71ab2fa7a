"""B200-native multinomial resampling (arXiv 2604.01356), drop-in for ``dacresample``.

Same public names as /root/reference/pkg/src/dacresample/__init__.py:12-52
for the resampling path: random streams and sorted uniforms, weight tables,
and the binary / Carpenter-Clifford-Fearnhead / divide-and-conquer samplers,
all computed by hand-written sm_100a kernels in ``libdrs.so`` through a
ctypes C ABI (include/drs.h).  Weight-field generators (weightgen.py), the
timing harness and the CLI are outside this package's scope.

Beyond the reference: ``resample_batched`` (many independent filters in one
launch) and ``ShardedWeightTable`` / ``sharded_dac_sampler`` (one table split
over several GPUs with a single all-gather of shard totals).
"""

from .batched import BatchedStreams, resample_batched
from .cdf import WeightTable, build_weight_table, build_weight_table_from_log, upper_bound_search
from .randkit import DeviceRngStream, RngStream, sorted_uniforms, uniform_open
from .samplers import (
    OpStats,
    binary_sampler,
    ccf_match,
    ccf_sampler,
    dac_match,
    dac_sampler,
    linear_oracle,
    warm_kernels,
)
from .sharded import ShardedWeightTable, build_sharded_table, sharded_dac_sampler
from .verify import (chi_square_statistic, gather_states, histogram, resample_and_gather, verify_complexity,
                     verify_statistics)

__all__ = [
    "RngStream",
    "DeviceRngStream",
    "uniform_open",
    "sorted_uniforms",
    "WeightTable",
    "build_weight_table",
    "build_weight_table_from_log",
    "upper_bound_search",
    "OpStats",
    "linear_oracle",
    "binary_sampler",
    "ccf_match",
    "ccf_sampler",
    "dac_match",
    "dac_sampler",
    "warm_kernels",
    "resample_batched",
    "BatchedStreams",
    "ShardedWeightTable",
    "build_sharded_table",
    "sharded_dac_sampler",
    "gather_states",
    "resample_and_gather",
    "histogram",
    "chi_square_statistic",
    "verify_statistics",
    "verify_complexity",
]

__version__ = "0.1.0"
