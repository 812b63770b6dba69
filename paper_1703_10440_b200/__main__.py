"""``python -m paper_1703_10440_b200 {factor,bench} ...`` (cli.py)."""

from .cli import entry

entry()
