// detector oracle: filled in below
