from paper_2410_00161_b200.cache import *  # noqa: F401,F403
from paper_2410_00161_b200.cache import BlockTables, SlotHandle, UnifiedKVCache, append_kv, fragmentation, lookup_kv  # noqa: F401
