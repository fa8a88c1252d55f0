from paper_2410_00161_b200.attention import *  # noqa: F401,F403
from paper_2410_00161_b200.attention import AttentionConfig, dense_attention, gqa_attention, paged_attention  # noqa: F401
