"""TEST INFRASTRUCTURE ONLY: CPU oracle (restatement + compiled reference)."""
