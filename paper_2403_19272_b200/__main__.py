"""python -m paper_2403_19272_b200 simulate|verify|bench-ccd ... (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
