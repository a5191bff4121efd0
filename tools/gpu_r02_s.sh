#!/bin/bash
# r02 experiment: CTA start stagger (BSIM_EXP_STAGGER_CYC) -- co-resident CTAs out of phase
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out/stagger
for v in "" st3k st6k st9k "" st6k; do echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_step_bench.py --models quadruped,quadruped12,humanoid --envs 4096,16384 --prec fp32 2>&1 | grep us/control; done
