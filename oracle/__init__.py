"""CPU oracle (test infrastructure only): a NumPy restatement of the reference
densolve hot path, pinned to golden vectors from the reference itself.
Never imported by the product package paper_1511_07207_b200."""
