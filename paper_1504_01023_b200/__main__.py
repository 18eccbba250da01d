"""``python -m paper_1504_01023_b200 {verify,bench,tune,model,genmesh}`` (see ``cli.py``)."""

import sys

from .cli import main

sys.exit(main())
