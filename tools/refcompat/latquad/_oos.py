"""Out-of-scope names of the reference (symbolic algebra, transform
validation): present so imports resolve, unimplemented when called."""


def _missing(name):
    def f(*args, **kwargs):
        raise NotImplementedError(f"latquad.{name} is outside the GPU hot path (DESIGN.md §8)")
    f.__name__ = name
    return f


class NonCartesianStructureError(ValueError):
    pass


class TransformedIntegrand:
    def __init__(self, *args, **kwargs):
        raise NotImplementedError("TransformedIntegrand is outside the GPU hot path (DESIGN.md §8)")


bind = _missing("bind")
partial_sum = _missing("partial_sum")
substitute = _missing("substitute")
normalize = _missing("exprcore.normalize")
build_axis_grids = _missing("build_axis_grids")
forward_transform = _missing("forward_transform")
grid_completion = _missing("grid_completion")
inverse_substitution = _missing("inverse_substitution")
make_transformed_integrand = _missing("make_transformed_integrand")
