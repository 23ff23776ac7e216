"""Drop-in module aliases: after ``install()``, ``import meshfree`` and the
reference's submodule paths resolve to this package, so code (and tests)
written against the reference run unchanged on the B200 path.

    import paper_1912_13282_b200.compat as compat
    compat.install()
    from meshfree import NodeSet, find_closest_stencils          # this package
    from meshfree.approx.engines import RbfFd                     # this package
    from meshfree.drivers import run_heat_explicit                # this package

The layout mirrored is the reference's (pkg/src/meshfree/__init__.py:10-48,
geometry/__init__.py:1-6, approx/__init__.py:1-19): ``meshfree.geometry``
(``nodeset``, ``stencils``, ``fill``, ``shapes``, ``spacing``),
``meshfree.approx`` (``basis``, ``operators``, ``weights``, ``engines``),
``meshfree.storage``, ``meshfree.assembly``, ``meshfree.solve``,
``meshfree.drivers``, ``meshfree.errors``.  Names of the reference that lie
outside the hot path (boundary discretisation, studies, CLI, thread/backend
switches) exist as stubs that raise ``ConfigError`` when called,
so importing them does not fail.

A caller who keeps the reference installed for those parts can hand it over:

    import meshfree as reference                 # the CPU package
    compat.install(force=True, reference=reference)
    nodes = meshfree.discretize_boundary(shape, 0.05)   # reference geometry, returns THIS package's NodeSet
    nodes = meshfree.fill_interior(nodes, shape, 0.05)  # B200 from here on

``discretize_boundary``, ``grid_nodes`` and ``add_ghost_nodes`` then run in the
reference (host geometry, not on the hot path) with shapes and node sets
converted at the border; nothing else is routed there.
"""

from __future__ import annotations

import sys
import types

from .errors import ConfigError

_OUT_OF_SCOPE = {
    "meshfree.geometry": ("discretize_boundary", "add_ghost_nodes", "grid_nodes"),
    "meshfree.geometry.boundary": ("discretize_boundary", "add_ghost_nodes", "grid_nodes"),
    "meshfree": ("discretize_boundary", "add_ghost_nodes", "grid_nodes", "set_threads"),
    "meshfree.config": ("set_threads",),
}


def _stub(name):
    def missing(*args, **kwargs):
        raise ConfigError(f"{name} is outside the B200 hot path (boundary discretisation, studies, CLI and "
                          "thread switches stay with the reference package)")

    missing.__name__ = name
    return missing


def _module(name, sources, names=None):
    """A module object `name` exposing `names` (default: every public name) of `sources`."""
    mod = types.ModuleType(name)
    mod.__doc__ = f"alias of {', '.join(s.__name__ for s in sources)} (paper_1912_13282_b200.compat)"
    for src in sources:
        for key in (names if names is not None else getattr(src, "__all__", None) or
                    [k for k in vars(src) if not k.startswith("_")]):
            if hasattr(src, key) and not hasattr(mod, key):
                setattr(mod, key, getattr(src, key))
    for key in _OUT_OF_SCOPE.get(name, ()):
        if not hasattr(mod, key):
            setattr(mod, key, _stub(key))
    return mod


def backend_name() -> str:
    """The reference reports "numba" or "numpy" (config.py:60-78); here every kernel is CUDA."""
    return "cuda-sm_100a"


def _boundary_bridge(reference):
    """discretize_boundary / grid_nodes / add_ghost_nodes of the reference package,
    taking and returning this package's shapes and node sets."""
    from . import geometry
    from .nodeset import NodeSet

    rgeo = reference.geometry
    rshapes, rboundary = rgeo.shapes, rgeo.boundary

    def to_ref_shape(s):
        if isinstance(s, geometry.Ball):
            return rshapes.Ball(s.center, s.radius, tag=s.tag)
        if isinstance(s, geometry.Box):
            return rshapes.Box(s.lo, s.hi, tag=s.tag)
        if isinstance(s, geometry.ShapeUnion):
            return rshapes.ShapeUnion(to_ref_shape(s.a), to_ref_shape(s.b))
        if isinstance(s, geometry.ShapeDifference):
            return rshapes.ShapeDifference(to_ref_shape(s.a), to_ref_shape(s.b))
        if isinstance(s, geometry.Translated):
            return rshapes.Translated(to_ref_shape(s.inner), s.offset)
        if isinstance(s, geometry.Rotated):
            return rshapes.Rotated(to_ref_shape(s.inner), s.matrix)
        return s  # already a reference shape (or a user class with the same methods)

    def to_nodes(n):
        return NodeSet(n.positions, n.types, n.normals)

    def discretize_boundary(shape, h, seed: int = 0):
        return to_nodes(rboundary.discretize_boundary(to_ref_shape(shape), h, seed))

    def grid_nodes(*args, **kwargs):
        return to_nodes(rboundary.grid_nodes(*args, **kwargs))

    def add_ghost_nodes(nodes, h, tag: int = 0, which="boundary"):
        new, ghost_of = rboundary.add_ghost_nodes(rgeo.NodeSet(nodes.positions, nodes.types, nodes.normals), h, tag,
                                                  which)
        return to_nodes(new), ghost_of

    return {"discretize_boundary": discretize_boundary, "grid_nodes": grid_nodes, "add_ghost_nodes": add_ghost_nodes}


def install(name: str = "meshfree", *, force: bool = False, reference=None) -> types.ModuleType:
    """Register this package under the reference's module paths and return the root alias.

    Raises ConfigError if a different ``meshfree`` is already imported (unless force=True):
    silently shadowing the reference would hide which implementation ran.  With
    ``reference=<the imported CPU package>`` the three boundary-discretisation functions
    (out of scope here) are served by it; everything else stays this package."""
    import paper_1912_13282_b200 as pkg
    from . import approx, assembly, drivers, errors, geometry, nodeset, solve, stencils, storage

    present = sys.modules.get(name)
    if present is not None and getattr(present, "__b200_alias__", False):
        return present
    if present is not None and not force:
        raise ConfigError(f"a module named {name!r} is already imported from {getattr(present, '__file__', '?')}")

    root = _module(name, [pkg])
    root.__b200_alias__ = True
    root.backend_name = backend_name
    root.__path__ = []  # a package: submodule imports go through sys.modules
    geo = _module(f"{name}.geometry", [geometry, nodeset, stencils],
                  ["Ball", "Box", "ConstantSpacing", "LinearSpacing", "NodeSet", "Shape", "ShapeDifference",
                   "ShapeUnion", "as_spacing", "fill_interior", "find_closest_stencils"])
    geo.__path__ = []
    apx = _module(f"{name}.approx", [approx],
                  ["ConstantWeight", "Directional", "FirstDerivative", "Gaussian", "GaussianWeight", "Identity",
                   "InverseMultiquadric", "Laplacian", "MonomialBasis", "Multiquadric", "Operator", "OperatorSum",
                   "Polyharmonic", "RbfFd", "ScaledOperator", "SecondDerivative", "WeightedLeastSquares"])
    apx.__path__ = []
    cfg = _module(f"{name}.config", [], [])
    cfg.backend_name = backend_name
    subs = {
        f"{name}.geometry": geo,
        f"{name}.geometry.nodeset": nodeset,
        f"{name}.geometry.stencils": stencils,
        f"{name}.geometry.fill": geometry,
        f"{name}.geometry.shapes": geometry,
        f"{name}.geometry.spacing": geometry,
        f"{name}.geometry.boundary": _module(f"{name}.geometry.boundary", [], []),
        f"{name}.approx": apx,
        f"{name}.approx.basis": approx,
        f"{name}.approx.operators": approx,
        f"{name}.approx.weights": approx,
        f"{name}.approx.engines": approx,
        f"{name}.storage": storage,
        f"{name}.assembly": assembly,
        f"{name}.solve": solve,
        f"{name}.drivers": drivers,
        f"{name}.errors": errors,
        f"{name}.config": cfg,
    }
    if reference is not None:
        for key, fn in _boundary_bridge(reference).items():
            for mod in (root, geo, subs[f"{name}.geometry.boundary"]):
                setattr(mod, key, fn)
    sys.modules[name] = root
    for path, mod in subs.items():
        sys.modules[path] = mod
        parent, _, leaf = path.rpartition(".")
        setattr(sys.modules[parent], leaf, mod)
    return root


def uninstall(name: str = "meshfree") -> None:
    """Remove the aliases registered by install()."""
    if getattr(sys.modules.get(name), "__b200_alias__", False):
        for key in [k for k in sys.modules if k == name or k.startswith(name + ".")]:
            del sys.modules[key]
