"""Seeded synthetic workloads of BASELINE.json's configs (test / bench input only)."""
