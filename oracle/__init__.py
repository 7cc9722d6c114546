"""CPU parity oracle for the integral-image regularizer (test infrastructure only).

Not part of the product: see oracle/inim_oracle.c and oracle/oracle.py headers.
"""
