"""Python mirror of the reference exception hierarchy
(proj/include/hydro/errors.hpp:11-34): a located ``SimError`` and its five
subclasses, rebuilt from the C-ABI ``h2d_error`` record."""
from __future__ import annotations

H2D_OK, H2D_ERR_SIM, H2D_ERR_TANGLED, H2D_ERR_UNPHYSICAL = 0, 1, 2, 3
H2D_ERR_NEGMASS, H2D_ERR_CFL, H2D_ERR_ISOLATED = 4, 5, 6
H2D_ERR_INVALID, H2D_ERR_DEVICE, H2D_ERR_NOMEM = 100, 101, 102


class SimError(RuntimeError):
    """Runtime failure of the scheme with the offending cell/node and step."""

    def __init__(self, what: str, i: int = -1, j: int = -1, step: int = -1, in_step: bool = False):
        super().__init__(what)
        self.what, self.i, self.j, self.step, self.in_step = what, i, j, step, in_step
        self.partial = None

    def run_message(self, case_name: str) -> str:
        """The message run() re-throws for errors inside a step
        (harness.cpp:404-407)."""
        if self.in_step:
            return f"{self.what} [{case_name} step {self.step}]"
        return self.what


class TangledCellError(SimError):
    pass


class UnphysicalStateError(SimError):
    pass


class NegativeMassError(SimError):
    pass


class CflViolationError(SimError):
    pass


class IsolatedMixedCellError(SimError):
    pass


class DeviceError(RuntimeError):
    """CUDA runtime failure or invalid use of the ABI (not a reference error)."""

    def __init__(self, what: str, code: int = H2D_ERR_DEVICE):
        super().__init__(what)
        self.code = code


_KIND = {H2D_ERR_SIM: SimError, H2D_ERR_TANGLED: TangledCellError, H2D_ERR_UNPHYSICAL: UnphysicalStateError,
         H2D_ERR_NEGMASS: NegativeMassError, H2D_ERR_CFL: CflViolationError,
         H2D_ERR_ISOLATED: IsolatedMixedCellError}


def from_code(code: int, what: str) -> Exception:
    cls = _KIND.get(code)
    return cls(what) if cls else DeviceError(what, code)


def from_record(rec) -> Exception:
    what = rec.what.decode(errors="replace")
    cls = _KIND.get(rec.kind)
    if cls is None:
        return DeviceError(what or f"error {rec.kind}", rec.kind)
    return cls(what, rec.i, rec.j, rec.step, bool(rec.in_step))
