for c in 2 3 4 8; do for cw in 8 4; do echo "ctas=$c cw=$cw"; PPMOE_OG_CTAS=$c PPMOE_OG_FWD_CW=$cw timeout 120 python tools/micro.py 2>&1 | grep "owner gather"; done; done
