"""Seeded synthetic inputs shared by the oracle tests and the product path.

This package holds NONE of the method's arithmetic (no fluxes, no sweeps, no
coloring, no agglomeration).  It only builds meshes (topology + geometry,
computed once here and consumed identically by both sides) and initial
states.  See DESIGN.md "Input recipe".
"""
from .mesh import Mesh, FARFIELD, SLIP, NOSLIP, EXTRAP  # noqa: F401
from . import configs, state  # noqa: F401
