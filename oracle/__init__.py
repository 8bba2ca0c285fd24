"""TEST INFRASTRUCTURE ONLY: CPU parity oracle of the reference TWED path (see oracle.py)."""
