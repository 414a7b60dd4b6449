"""``python -m paper_2309_03912_b200 check|corpus ...`` (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
