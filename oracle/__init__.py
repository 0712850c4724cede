"""TEST INFRASTRUCTURE ONLY -- CPU parity checkers for the fbf filtering path.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this package. The product library
(paper_1811_02168_b200) never imports, links or executes anything here.
"""
