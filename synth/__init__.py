"""Seeded synthetic workloads shared by tests and bench (no method arithmetic)."""
