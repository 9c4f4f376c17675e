"""Harness-side synthetic workloads (not product code).

Kept outside the product package so that benchmark arms and checkers can build
inputs without importing ``paper_2302_07411_b200`` (whose import maps
``libcve_b200.so``): the reference arm of ``bench.py`` must load only the
reference's own library.
"""
