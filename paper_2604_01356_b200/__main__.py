"""python -m paper_2604_01356_b200 {sample,verify,bench} (cli.py)."""

import sys

from .cli import main

sys.exit(main())
