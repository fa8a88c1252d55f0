from paper_2410_00161_b200.engine import *  # noqa: F401,F403
from paper_2410_00161_b200.budget import budget_to_blocks, per_sequence_budget  # noqa: F401
