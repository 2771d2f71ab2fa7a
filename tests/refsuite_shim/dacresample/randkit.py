"""dacresample.randkit -> paper_2604_01356_b200.randkit (test shim)."""

from paper_2604_01356_b200.randkit import *  # noqa: F401,F403
from paper_2604_01356_b200.randkit import RngStream, sorted_uniforms, uniform_open  # noqa: F401
