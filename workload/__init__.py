"""Input-side workload generator (synthetic BASELINE systems, snapshot bundles): libfp_workload.so."""
