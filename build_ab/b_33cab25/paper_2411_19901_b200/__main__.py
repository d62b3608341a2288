"""``python -m paper_2411_19901_b200 run|bench|convert ...`` (cli.py)."""
import sys

from .cli import main

sys.exit(main())
