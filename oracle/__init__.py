"""CPU oracle -- TEST INFRASTRUCTURE ONLY (see tl_oracle.py header).

Importable only from tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs. The product package never imports it.
"""
