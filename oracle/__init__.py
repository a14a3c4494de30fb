"""Test-only oracles (CPU restatements / reference-generated fixtures).
Never imported by the product package."""
