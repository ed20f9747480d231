"""python -m paper_2207_11620_b200 <subcommand> ... (the reference's `neuralvol` entry point)."""
import sys

from .cli import main

sys.exit(main())
