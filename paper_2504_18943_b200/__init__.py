"""B200-native drop-in for the reference's LTLf enumeration path.

Same public names as the reference package ``ltlsynth`` (reference
``pkg/src/ltlsynth/__init__.py:9-76``) for everything on or next to the
enumeration hot path; the enumeration itself runs in hand-written sm_100a
CUDA behind the C-ABI declared in ``include/ltlsynth_b200.h``.
"""

from .formulas import (
    DEFAULT_OPERATORS,
    OPERATOR_NAMES,
    And,
    Atom,
    Formula,
    Future,
    Next,
    Not,
    Or,
    Until,
    cost,
    parse_formula,
    to_text,
)
from .semantics import sat, separates_by_sat
from .traces import (
    Alphabet,
    InfeasibleSpecificationError,
    Layout,
    SpecError,
    SpecFormatError,
    Specification,
    Trace,
    atom_bitvectors,
    parse_specification,
    serialize_specification,
    smallest_lane_dtype,
    spec_from_steps,
    step_trace,
    validate_feasible,
    word_trace,
)

__version__ = "0.1.0"
