"""Test infrastructure: CPU oracle of the reference Mapper hot path.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline arm. See mapper_oracle.py for the restatement and its citations.
"""
