"""B200-native Flash-MaxSim operator (sm_100a), a drop-in for the reference `maxsim` path."""
