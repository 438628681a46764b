"""CPU oracle package (test infrastructure only; see oracle/emst_oracle.c)."""
