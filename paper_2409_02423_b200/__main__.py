"""python -m paper_2409_02423_b200 {run,sweep,codec-bench,validate} (cli.py)."""
import sys

from .cli import main

sys.exit(main())
