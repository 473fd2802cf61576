"""``python -m paper_2504_18943_b200 synth|check ...`` (see cli.py)."""
from .cli import entry_point

entry_point()
