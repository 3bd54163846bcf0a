"""``python -m paper_2004_08962_b200 recon --config run.json`` (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
