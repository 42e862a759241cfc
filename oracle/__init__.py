"""Oracle package — TEST INFRASTRUCTURE ONLY (tests/, smoke(), bench cpu_baseline)."""
