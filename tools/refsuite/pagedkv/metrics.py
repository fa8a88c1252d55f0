from paper_2410_00161_b200.metrics import *  # noqa: F401,F403
from paper_2410_00161_b200.metrics import (MetricConfig, MetricsStore, accumulate_decode, full_metrics,  # noqa: F401
                                           prompt_metrics, window_metrics)
