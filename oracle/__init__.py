"""Plain CPU oracle (test infrastructure only; see oracle/cp_oracle.c)."""
