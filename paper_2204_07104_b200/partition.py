"""Compatibility alias: ``sptucker.partition`` names."""
from .schedule import (PartitionPlan, RoundSchedule, build_partition, round_schedule,  # noqa: F401
                       schedule_text)
