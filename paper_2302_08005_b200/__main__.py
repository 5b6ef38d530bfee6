"""`python -m paper_2302_08005_b200 ...`: the slapo CLI surface (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
