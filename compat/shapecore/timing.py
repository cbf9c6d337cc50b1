"""shapecore.timing: StageTimings (B200 package)."""
from paper_2510_02894_b200.timing import StageTimings  # noqa: F401
