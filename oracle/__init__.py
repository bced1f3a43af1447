"""TEST INFRASTRUCTURE ONLY: CPU restatement of the reference hot path.

Imported by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs;
never by the product package."""
