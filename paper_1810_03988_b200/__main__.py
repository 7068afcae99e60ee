"""python -m paper_1810_03988_b200 stitch|extract|bench ... (the lorbpano CLI)."""
import sys

from .cli import main

sys.exit(main())
