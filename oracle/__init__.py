"""Test-infrastructure oracle (CPU restatement of the reference path).

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU legs.
"""
