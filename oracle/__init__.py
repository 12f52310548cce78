"""Test-only CPU checkers (see oracle/heoracle.h)."""
