#!/bin/bash
# re-entry check of HEAD: GPU suite + smoke + bench
bash tools/gpu_round.sh tests bench
