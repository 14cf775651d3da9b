#!/bin/bash
# chain-priority A/B, then the round's final evidence pass (default settings)
bash tools/runs/gpu_r2e_prio.sh
bash tools/runs/gpu_r2e_final.sh
