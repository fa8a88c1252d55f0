from paper_2410_00161_b200.block_manager import *  # noqa: F401,F403
from paper_2410_00161_b200.block_manager import BlockManager, blocks_needed_prefill  # noqa: F401
from paper_2410_00161_b200.engine import preempt_select  # noqa: F401
