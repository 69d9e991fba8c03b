"""python -m paper_2204_07921_b200 <command> ... (the CLI harness, cli.py)."""

from .cli import main

main()
