#!/bin/bash
# round-2 GPU session 15b (4 GPUs): sessions 15 + 16 in one call
bash tools/sessions/r2_session15.sh
bash tools/sessions/r2_session16.sh
