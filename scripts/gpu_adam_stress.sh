#!/bin/bash
for pdl in 1 0 1 0; do ASTRA_PDL=$pdl timeout 600 python scripts/adam_stress.py 150 2>&1 | tail -1; done
