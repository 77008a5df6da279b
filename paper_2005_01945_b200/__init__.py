"""B200-native TFHE gate-evaluation engine behind the `encirc` GateEngine API."""
