"""Error vocabulary of the reference boundary (types.hpp:16-46)."""


class Error(RuntimeError):
    pass


class LevelUnderflow(Error):
    pass


class InvalidTarget(Error):
    pass


class ShapeMismatch(Error):
    pass


class LayoutMismatch(Error):
    pass


class CacheFull(Error):
    pass


class CacheEmpty(Error):
    pass


class DomainViolation(Error):
    pass
