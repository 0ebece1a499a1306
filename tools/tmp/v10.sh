timeout 900 python -m pytest tests -m gpu -x -q -k "pcg_iteration_sequences or stored_quadrature or pcg_error" 2>&1 | tail -15
