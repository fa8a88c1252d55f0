from paper_2410_00161_b200.errors import *  # noqa: F401,F403
