"""CPU oracle of the CWTH path -- test infrastructure only (see oracle.py)."""
