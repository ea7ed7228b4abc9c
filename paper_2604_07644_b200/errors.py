"""Exception classes with the reference's names, bases and messages.

lqr.py:31-40 (IllConditionedCombineError, SingularStageError,
CacheInvalidatedError), sqp.py:23 (DivergenceError), sls.py:29
(RobustInfeasibleError).
"""


class IllConditionedCombineError(ArithmeticError):
    pass


class SingularStageError(ArithmeticError):
    pass


class CacheInvalidatedError(RuntimeError):
    pass


class DivergenceError(RuntimeError):
    pass


class RobustInfeasibleError(RuntimeError):
    pass
