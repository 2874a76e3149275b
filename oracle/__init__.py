"""ORACLE package -- test infrastructure only (see oracle/README.md).

Importable only from tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.
"""
