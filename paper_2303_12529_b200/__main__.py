"""`python -m paper_2303_12529_b200 <command> ...`: the CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())
