"""python -m paper_2008_03095_b200 select|evaluate|cdf ... (cli.py)."""
import sys

from .cli import main

sys.exit(main())
