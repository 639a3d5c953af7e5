"""`python -m paper_2405_19493_b200 ...`: the gausszig-style CLI on the B200 engine."""
from .cli import entrypoint

entrypoint()
