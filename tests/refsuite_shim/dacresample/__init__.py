"""``dacresample`` name shim over the GPU package (test infrastructure only).

Lets the reference's own test modules (/root/reference/pkg/tests, copied
untracked into baseline/_ref/refsuite by scripts/run_reference_suite.py) run
unchanged against paper_2604_01356_b200: the in-scope modules cdf, randkit
and samplers map onto the GPU package; bench, weightgen and cli are outside
this package's scope and are not provided.
"""

from paper_2604_01356_b200 import *  # noqa: F401,F403
from paper_2604_01356_b200 import __all__, __version__  # noqa: F401
