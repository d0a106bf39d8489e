"""Complex walk (placeholder until the c128 kernels land)."""


def complex_walk_total(m, devices=None):
    raise NotImplementedError("complex kernels not built yet")


def complex_ranges(m, spans, exact=None, devices=None):
    raise NotImplementedError("complex kernels not built yet")
