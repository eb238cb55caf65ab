"""Bench / test workloads (synthetic scenarios and reference-generated trace
window statistics). Not part of the product package."""
