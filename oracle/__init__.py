"""CPU checkers for the B200 hot path (TEST INFRASTRUCTURE ONLY)."""
