cd $GRAFT_REPO_ROOT
for e in '' 'CMG_ENERGY_TARGET=512' 'CMG_ENERGY_TARGET=2048' 'CMG_ENERGY_TARGET=256' 'CMG_ENERGY_CTAS=1184'; do env $e python tools/stamps_report.py fast float64 | grep -E "energy|per cycle" | tr '\n' ' '; echo " <- $e"; done
