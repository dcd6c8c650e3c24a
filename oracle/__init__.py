"""CPU oracle for the charging-station step — TEST INFRASTRUCTURE ONLY.

Imported by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
reference legs as the checker; the product package never imports it.
"""
