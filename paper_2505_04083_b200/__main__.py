"""python -m paper_2505_04083_b200 {preprocess,train,rank-configs} (cli.py)."""
import sys

from .cli import main

sys.exit(main())
