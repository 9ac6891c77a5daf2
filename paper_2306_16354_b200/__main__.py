"""``python -m paper_2306_16354_b200 <subcommand>``: the parlink-compatible CLI (cli.py)."""

import sys

from .cli import main

sys.exit(main())
