for k in 1 2 4 8; do echo "parts $k"; VXG_H2D_PARTS=$k python tools/probe_e2e.py; done
