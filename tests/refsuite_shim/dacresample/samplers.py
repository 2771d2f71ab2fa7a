"""dacresample.samplers -> paper_2604_01356_b200.samplers (test shim)."""

from paper_2604_01356_b200.samplers import *  # noqa: F401,F403
from paper_2604_01356_b200.samplers import (  # noqa: F401
    OpStats,
    binary_sampler,
    ccf_match,
    ccf_sampler,
    dac_match,
    dac_sampler,
    linear_oracle,
    warm_kernels,
)
from paper_2604_01356_b200.cdf import WeightTable, upper_bound_search  # noqa: F401
from paper_2604_01356_b200.randkit import RngStream, sorted_uniforms  # noqa: F401
