"""CPU oracle of the GSFusion rasterizer hot path -- TEST INFRASTRUCTURE ONLY.

Importable by tests/, __graft_entry__.smoke() and bench.py's CPU baseline legs;
never by the product package.  See gsref.cpp for the definitions.
"""
