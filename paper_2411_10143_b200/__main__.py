"""``python -m paper_2411_10143_b200 <command>`` — the reference CLI on B200 (cli.py)."""
import sys

from .cli import main

sys.exit(main())
