"""``python -m paper_2203_08966_b200`` == the ``nbsim`` console script (harness.main)."""

import sys

from .harness import main

sys.exit(main())
