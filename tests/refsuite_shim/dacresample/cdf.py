"""dacresample.cdf -> paper_2604_01356_b200.cdf (test shim)."""

from paper_2604_01356_b200.cdf import *  # noqa: F401,F403
from paper_2604_01356_b200.cdf import WeightTable, build_weight_table, upper_bound_search  # noqa: F401
