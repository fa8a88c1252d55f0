from paper_2410_00161_b200.compression import *  # noqa: F401,F403
