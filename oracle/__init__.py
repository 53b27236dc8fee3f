"""CPU oracle — TEST INFRASTRUCTURE ONLY (see seed_oracle.py header)."""
from .seed_oracle import *  # noqa: F401,F403
