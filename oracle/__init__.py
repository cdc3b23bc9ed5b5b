"""CPU oracle (test infrastructure only) — see ttb_oracle.py's header."""
