"""TEST INFRASTRUCTURE ONLY: CPU oracle restating the reference `axemu` path.

See oracle/axemu_oracle.py.  Importable only from tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs.
"""
