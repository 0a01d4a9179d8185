class ContractError(ValueError):
    """An operation was called with arguments that violate its contract.

    Same name and base class as the reference's tierkv.errors.ContractError
    (errors.py:1-2), so callers catching ValueError keep working.
    """
