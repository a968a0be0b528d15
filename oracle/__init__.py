"""CPU oracle -- TEST INFRASTRUCTURE ONLY (see oracle/albref.h)."""
