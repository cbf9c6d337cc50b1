"""shapecore.errors: the B200 package's exception hierarchy (same classes)."""
from paper_2510_02894_b200.errors import *  # noqa: F401,F403
