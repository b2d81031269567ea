"""`python -m paper_1603_08109_b200 ...`: the command-line front end (cli.py)."""

from .cli import main

main()
