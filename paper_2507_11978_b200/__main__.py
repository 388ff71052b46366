"""`python -m paper_2507_11978_b200 run ...` = the B200 artifact runner."""
import sys

from .runner import main

sys.exit(main())
