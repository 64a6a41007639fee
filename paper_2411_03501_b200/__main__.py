"""``python -m paper_2411_03501_b200 solve|selftest ...`` -- the ``hjls`` command (cli.py:256-296)."""
import sys

from .cli import main

sys.exit(main())
